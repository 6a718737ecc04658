set -u
AB_NODEFAULT=1 bash tools/gpu_ab.sh 4 f64 k512 k256 2>&1 | grep -v rep3
AB_NODEFAULT=1 bash tools/gpu_ab.sh 2 f64 whatif_nostore 2>&1 | grep -v rep3
for V in k512 k256; do ZSB_LIB_VARIANT=$V timeout -s KILL 300 python tools/variant_check.py 2>&1 | tail -n 3; done
