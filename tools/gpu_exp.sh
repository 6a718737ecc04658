mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
for V in "ZSB_SW16_ABOVE=1024" "ZSB_SW16_ABOVE=512" "ZSB_SW16_ABOVE=512 ZSB_TILES_PER_SM=2"; do
  T=$(echo $V | tr ' =' '__')
  env $V $CMD > gpurun_out/exp_$T.log 2>&1 && \
  env $V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
      --log-file gpurun_out/exp_$T.csv $CMD > /dev/null 2>&1
  echo "$V rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/exp_$T.log)"
done
