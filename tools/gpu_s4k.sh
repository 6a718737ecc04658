set -u
O=gpurun_out; mkdir -p $O
ZSB_LIB_VARIANT=ft512 timeout -s KILL 600 python tools/variant_check.py > $O/s4k_check.log 2>&1; echo "check rc=$?"; grep -c ok $O/s4k_check.log; grep -i "mismatch\|violations\|error" $O/s4k_check.log | head
AB_NODEFAULT=1 bash tools/gpu_ab.sh 4 noteam ft512 2>&1 | grep -v rep3
AB_NODEFAULT=1 bash tools/gpu_ab.sh 2 noteam ft512 2>&1 | grep -v rep3
