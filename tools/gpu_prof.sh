# launch list + full profile of the hot kernels (1 GPU). Plain run first, same args.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_finish|k_classify|k_hist" -s 8 -c 4 \
    -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
