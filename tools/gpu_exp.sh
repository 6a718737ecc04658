# usage: bash tools/gpu_exp.sh "ENV1=a ENV2=b" "ENV1=c" ...   (one bench + launch list per variant)
mkdir -p gpurun_out
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators"
for V in "$@"; do
  T=$(echo "$V" | tr ' =' '__')
  env $V $CMD > gpurun_out/exp_$T.log 2>&1
  echo "$V rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/exp_$T.log)"
  env $V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
      --log-file gpurun_out/exp_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /dev/null 2>&1
done
