set -u
O=gpurun_out; mkdir -p $O
ZSB_LIB_VARIANT=f64 timeout -s KILL 600 python tools/variant_check.py > $O/s4h_check.log 2>&1; echo "check rc=$?"; grep -c ok $O/s4h_check.log; grep -i "mismatch\|violations" $O/s4h_check.log
AB_NODEFAULT=1 bash tools/gpu_ab.sh 4 noruns f64 2>&1 | grep -v rep3
AB_NODEFAULT=1 bash tools/gpu_ab.sh 2 noruns f64 2>&1 | grep -v rep3
