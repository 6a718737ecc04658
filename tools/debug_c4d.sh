for i in 1 2 3; do
echo "== 3e7 run $i"; timeout 300 python tools/debug_c4.py 30000000 fitted 2>&1 | grep -E "violations|unsorted"
done
echo "== 1e8"; timeout 300 python tools/debug_c4.py 100000000 fitted 2>&1 | grep -E "violations|unsorted|stats"
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
