n=30000000
echo "== default"; ZSB_DEBUG=1 timeout 300 python tools/debug_c4.py $n fitted 2>&1 | grep -E "level 3|violations|unsorted"
echo "== fin_ins 100000"; ZSB_FIN_INS=100000 timeout 300 python tools/debug_c4.py $n fitted 2>&1 | grep -E "violations|unsorted"
echo "== k1max 256"; ZSB_K1MAX=256 ZSB_DEBUG=1 timeout 300 python tools/debug_c4.py $n fitted 2>&1 | grep -E "level|violations|unsorted"
echo "== tiles1"; ZSB_TILES_PER_SM=1 timeout 300 python tools/debug_c4.py $n fitted 2>&1 | grep -E "violations|unsorted"
