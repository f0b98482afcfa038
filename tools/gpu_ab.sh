# A/B of two library builds (ab/old.so, ab/new.so) on one box: config #3
# breakdown and variant A, alternating.
mkdir -p gpurun_out
for r in 1 2; do
  for v in old new; do
    GPUOS_LIB=ab/$v.so timeout 600 python tools/hybrid_breakdown.py > gpurun_out/ab_hb_${v}_$r.txt 2>&1
    echo "$v $r hb rc=$?"; head -2 gpurun_out/ab_hb_${v}_$r.txt | cut -c1-200
    GPUOS_LIB=ab/$v.so timeout 900 python tools/hybrid_variants.py --only A --reps 2 > gpurun_out/ab_hv_${v}_$r.txt 2>&1
    echo "$v $r hv rc=$?"; grep -o '"p99_vs_alone": [0-9.]*\|"throughput_vs_static": [0-9.]*' gpurun_out/ab_hv_${v}_$r.txt | tr '\n' ' '; echo
  done
done
