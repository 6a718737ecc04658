set -u
O=gpurun_out; mkdir -p $O
B="python bench.py --no-cpu-baseline --no-e2e --no-comparators --no-extras"
for C in 4 2; do
  ZSB_LIB_VARIANT=prof timeout -s KILL 300 $B --config $C --steps 3 --warmup 3 > $O/s4c_prof_c$C.log 2>&1; echo "prof c$C rc=$?"
  grep -a "zsb\]" $O/s4c_prof_c$C.log | tail -n 2
done
AB_NODEFAULT=1 bash tools/gpu_ab.sh 2 f64 nostore norank 2>&1 | grep -v rep3
AB_NODEFAULT=1 bash tools/gpu_ab.sh 4 f64 norank 2>&1 | grep -v rep3
