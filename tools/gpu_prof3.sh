mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_finish|k_hist|k_moments" -s 10 -c 6 \
    -o gpurun_out/prof_r1c $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
