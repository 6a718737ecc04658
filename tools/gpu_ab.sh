# A/B: bench the default lib and each variant (ZSB_LIB_VARIANT) alternately, 3 times each.
# usage: bash tools/gpu_ab.sh CONFIG variant1 variant2 ...
mkdir -p gpurun_out
C=$1; shift
B="python bench.py --no-cpu-baseline --no-e2e --no-comparators --no-extras --steps 20 --warmup 5 --config $C"
for rep in 1 2 3; do
  for V in ${AB_NODEFAULT:+} ${AB_NODEFAULT:-default} "$@"; do
    [ "$V" = 1 ] && continue
    if [ "$V" = default ]; then E=""; else E="ZSB_LIB_VARIANT=$V"; fi
    env $E timeout -s KILL 300 $B > gpurun_out/ab_${V}_$rep.log 2>&1
    echo "$V c$C rep$rep: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${V}_$rep.log | head -1) $(grep -o '"phases_ms_per_step": {[^}]*}' gpurun_out/ab_${V}_$rep.log)"
  done
done
