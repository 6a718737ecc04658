mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_finish" -s 6 -c 3 \
    -o gpurun_out/prof_r1b $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
