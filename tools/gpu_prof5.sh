mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_finish" -s 4 -c 2 \
    -o gpurun_out/prof_fin6 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
