set -u
O=gpurun_out; mkdir -p $O
export ZSB_LIB_VARIANT=${1:-f64}
if [ ! -f /tmp/s4f_full_c4.ncu-rep ]; then
python tools/prof_sort.py --config 4 > $O/s4f_plain.log 2>&1 || exit 1
timeout -s KILL 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_scatter|k_finish|k_hist" -o /tmp/s4f_full_c4 python tools/prof_sort.py --config 4 > $O/s4f_ncu.log 2>&1; echo rc=$?
fi
ncu -i /tmp/s4f_full_c4.ncu-rep --page source --csv --print-source sass -k regex:k_scatter > $O/s4g_scatter_sass.csv 2>/dev/null
ncu -i /tmp/s4f_full_c4.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_scatter > $O/s4g_scatter_src.csv 2>/dev/null
ncu -i /tmp/s4f_full_c4.ncu-rep --page source --csv --print-source sass -k regex:k_finish > $O/s4g_finish_sass.csv 2>/dev/null
ncu -i /tmp/s4f_full_c4.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_finish > $O/s4g_finish_src.csv 2>/dev/null
ls -la $O
