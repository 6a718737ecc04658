# Produces the evidence committed under profiles/: bench line, per-kernel launch
# list (device time + DRAM bytes), one `ncu --set full` capture of the hot kernels.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators"
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > gpurun_out/${TAG}_gpu.txt
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_level1_map|k_hist|k_scatter|k_classify|k_finish" -s 12 -c 6 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?"
# the larger single-GPU workloads (C4 = 1e8 skewed float64, X9 = 1e9 uniform int64), bench lines only
for C in 4 9; do
  timeout -s KILL 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-comparators > gpurun_out/${TAG}_bench_c$C.json 2> gpurun_out/${TAG}_bench_c$C.err
  echo "bench c$C rc=$?"
done
