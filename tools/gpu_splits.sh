# Config #3 under different decode GEMV K splits (QKV, O, gate-up, down).
mkdir -p gpurun_out
for r in 1 2; do
  for sp in 3,4,1,4 3,4,3,4 3,4,2,4; do
    timeout 600 python tools/hybrid_breakdown.py --splits $sp > gpurun_out/sp_hb_${sp}_$r.txt 2>&1
    echo "$sp $r hb rc=$?"; head -2 gpurun_out/sp_hb_${sp}_$r.txt | cut -c1-110; grep "gemv_bf16 (28672" gpurun_out/sp_hb_${sp}_$r.txt
    timeout 900 python tools/hybrid_variants.py --only A --reps 3 --splits $sp > gpurun_out/sp_hv_${sp}_$r.txt 2>&1
    echo "$sp $r hv rc=$?"; grep -o '"p99_vs_alone": [0-9.]*\|"throughput_vs_static": [0-9.]*' gpurun_out/sp_hv_${sp}_$r.txt | tr '\n' ' '; echo
  done
done
