# Diagnostics: finish/scatter phase profile on C2, per-level log + timing on C4 and X9,
# launch list of one C4 sort.
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e --no-comparators"
ZSB_FIN_PROFILE=1 timeout -s KILL 300 $B --steps 3 --warmup 3 > gpurun_out/d_c2prof.log 2>&1; echo "c2prof rc=$?"
grep -a "zsb\]" gpurun_out/d_c2prof.log | tail -4
for C in 3 4 9; do
  ZSB_DEBUG=1 timeout -s KILL 600 $B --config $C --steps 5 --warmup 3 > gpurun_out/d_c$C.log 2>&1; echo "c$C rc=$?"
  grep -a "level" gpurun_out/d_c$C.log | tail -6
  tail -1 gpurun_out/d_c$C.log | grep -o '"ms_per_step": [0-9.]*\|"phases_ms_per_step": {[^}]*}'
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/d_c4_launches.csv $B --config 4 --steps 1 --warmup 3 > /dev/null 2>&1; echo "ncu rc=$?"
