# Session check: GPU tests, smoke, default bench, phase profiles (prof variant) on C4 and C2.
set -u
O=gpurun_out; mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/s4a_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 $O/s4a_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s4a_smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > $O/s4a_bench.json 2> $O/s4a_bench.err; echo "bench rc=$?"
B="python bench.py --no-cpu-baseline --no-e2e --no-comparators --no-extras"
for C in 4 2; do
  ZSB_LIB_VARIANT=prof timeout -s KILL 300 $B --config $C --steps 3 --warmup 3 > $O/s4a_prof_c$C.log 2>&1; echo "prof c$C rc=$?"
  grep -a "zsb\]" $O/s4a_prof_c$C.log | tail -n 12
done
