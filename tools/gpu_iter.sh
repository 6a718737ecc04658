# test + bench + per-kernel launch list (dram bytes) for a few tilings
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/bench.log
for V in "ZSB_TILES_PER_SM=2" "ZSB_TILES_PER_SM=1 ZSB_K1MAX=4096" "ZSB_TILES_PER_SM=1 ZSB_K1MAX=2048"; do
  T=$(echo $V | tr ' =' '__')
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators"
  env $V $CMD > gpurun_out/plain_$T.log 2>&1 && \
  env $V ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/launches_$T.csv $CMD > /dev/null 2>&1
  echo "$V rc=$?"
done
