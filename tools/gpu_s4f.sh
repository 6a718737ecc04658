set -u
O=gpurun_out; mkdir -p $O
export ZSB_LIB_VARIANT=${1:-f64}
python tools/prof_sort.py --config 4 > $O/s4f_plain.log 2>&1 || exit 1
timeout -s KILL 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_scatter|k_finish|k_hist" -o /tmp/s4f_full_c4 python tools/prof_sort.py --config 4 > $O/s4f_ncu.log 2>&1; echo rc=$?
python tools/ncu_key.py /tmp/s4f_full_c4.ncu-rep > $O/s4f_key.txt 2>&1
ncu -i /tmp/s4f_full_c4.ncu-rep --page raw --csv > $O/s4f_raw.csv 2>/dev/null
for K in "k_scatter<1, 4, 16" "k_scatter<1, 4, 8" "k_finish"; do
  T=$(echo "$K" | tr -dc 'a-z0-9_')
  python tools/ncu_src.py /tmp/s4f_full_c4.ncu-rep "$K" 45 > $O/s4f_src_$T.txt 2>&1
  python tools/ncu_inst.py /tmp/s4f_full_c4.ncu-rep "$K" 40 stall > $O/s4f_sass_$T.txt 2>&1
done
ls -la $O
