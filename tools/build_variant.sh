# usage: bash tools/build_variant.sh NAME "-DFLAG=.. ..."  -> paper_2605_14419_b200/libzsort_b200_NAME.so
set -e
P=paper_2605_14419_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr $2 -I include -o $P/libzsort_b200_$1.so $P/csrc/zsort_b200.cu 2>&1 | grep -i error || true
ls -la $P/libzsort_b200_$1.so
