# Round-2 evidence run on one B200: GPU tests, smoke, the default bench (C4),
# the C4 ncu launch list + one --set full capture of a whole sort, and
# compute-sanitizer over a C1-sized workload.  Usage: tools/gpu_round2.sh TAG [skip-tests]
set -u
TAG=${1:-r02a}
SKIP=${2:-}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem,memory.total --format=csv > $O/${TAG}_gpu.txt
python -c "import paper_2605_14419_b200._lib as l; l.load(auto_build=False); print(l.load().zsb_version())" > $O/${TAG}_version.txt 2>&1
if [ -z "$SKIP" ]; then
  timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?"
  timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
  echo "smoke rc=$?"
fi
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench rc=$?"
timeout -s KILL 600 python tools/prof_sort.py --config 4 > $O/${TAG}_plain.log 2>&1 && \
timeout -s KILL 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/${TAG}_launches_c4.csv python tools/prof_sort.py --config 4 > $O/${TAG}_ncu_l.log 2>&1
echo "launch list rc=$?"
timeout -s KILL 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -o $O/${TAG}_full_c4 python tools/prof_sort.py --config 4 > $O/${TAG}_ncu_full.log 2>&1
echo "full rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > $O/${TAG}_san_${tool}.log 2>&1
  echo "sanitizer $tool rc=$?"
done
