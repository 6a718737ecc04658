set -u
O=gpurun_out; mkdir -p $O
ZSB_LIB_VARIANT=f64 timeout -s KILL 600 python tools/variant_check.py > $O/s4b_check.log 2>&1; echo "check rc=$?"; tail -n 10 $O/s4b_check.log
AB_NODEFAULT=1 bash tools/gpu_ab.sh 4 base f64 smallonly looponly
AB_NODEFAULT=1 bash tools/gpu_ab.sh 2 base f64
