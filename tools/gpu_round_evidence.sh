# Final-state evidence: GPU tests, smoke, the default bench (C4), launch list with DRAM bytes of one C4 sort.
set -u
TAG=${1:-r02bb}
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem,memory.total --format=csv > $O/${TAG}_gpu.txt
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 $O/${TAG}_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"; tail -n 3 $O/${TAG}_bench.err
timeout -s KILL 600 python tools/prof_sort.py --config 4 > $O/${TAG}_plain.log 2>&1 && \
timeout -s KILL 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/${TAG}_launches_c4.csv python tools/prof_sort.py --config 4 > $O/${TAG}_ncu_l.log 2>&1
echo "launch list rc=$?"
