set -u
O=gpurun_out; mkdir -p $O
ZSB_LIB_VARIANT=f64 timeout -s KILL 600 python tools/variant_check.py > $O/s4e_check.log 2>&1; echo "check rc=$?"; grep -c ok $O/s4e_check.log; grep -i "mismatch\|violations" $O/s4e_check.log
AB_NODEFAULT=1 bash tools/gpu_ab.sh 4 f64 sk16 2>&1 | grep -v rep3
ZSB_LIB_VARIANT=prof timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --no-comparators --no-extras --config 4 --steps 3 --warmup 3 2>&1 | grep -a "zsb\]" | tail -n 2
