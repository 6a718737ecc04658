for n in 3000000 10000000 30000000; do
  echo "== n=$n"; ZSB_DEBUG=1 timeout 300 python tools/debug_c4.py $n fitted 2>&1 | grep -E "level|stats|violations|unsorted|permutation"
done
