# One `ncu --set full` capture of a C4 sort (hot kernels), summarised on the box into text files small
# enough to travel back (the .ncu-rep is ~70 MB): per-launch key metrics and stall ratios, instructions
# and stall samples per source line, shared-memory wavefronts per source line.
# usage: bash tools/gpu_ncu_full_c4.sh [LIB_VARIANT] [TAG]      (run under gpurun, one GPU)
set -u
O=gpurun_out; mkdir -p $O
[ -n "${1:-}" ] && export ZSB_LIB_VARIANT=$1
TAG=${2:-ncu_c4}
python tools/prof_sort.py --config 4 > $O/${TAG}_plain.log 2>&1 || exit 1
timeout -s KILL 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_scatter|k_finish|k_hist" -o /tmp/${TAG}_full python tools/prof_sort.py --config 4 > $O/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_key.py /tmp/${TAG}_full.ncu-rep > $O/${TAG}_key.txt 2>&1
python tools/ncu_lines.py /tmp/${TAG}_full.ncu-rep k_scatter 60 | cut -c1-170 > $O/${TAG}_lines_scatter.txt 2>&1
python tools/ncu_lines.py /tmp/${TAG}_full.ncu-rep k_finish 70 | cut -c1-170 > $O/${TAG}_lines_finish.txt 2>&1
python tools/ncu_smem.py /tmp/${TAG}_full.ncu-rep k_scatter 28 | cut -c1-200 > $O/${TAG}_smem_scatter.txt 2>&1
ls -la $O
