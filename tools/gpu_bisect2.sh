# Half A of the reverted handoff change (ab/A.so) vs the committed build:
# decode token A/B, then more of the split-K stress run and the bench's config runs on A.
mkdir -p gpurun_out
for r in 1 2; do
  for v in base A; do
    GPUOS_LIB=ab/$v.so timeout 600 python tools/hybrid_breakdown.py > gpurun_out/bis2_hb_${v}_$r.txt 2>&1
    echo "$v $r hb rc=$?"; head -2 gpurun_out/bis2_hb_${v}_$r.txt | cut -c1-100
  done
done
for i in $(seq 1 10); do
  GPUOS_LIB=ab/A.so timeout 300 python tools/hybrid_variants.py --only A --reps 3 --splits 3,4,3,4 > gpurun_out/bis2_A_$i.txt 2>&1
  echo "A $i rc=$? $(grep -o 'GpuosError.*' gpurun_out/bis2_A_$i.txt | cut -c1-150)"
done
GPUOS_LIB=ab/A.so timeout 900 python tools/hang_hunt2.py 2 > gpurun_out/bis2_hh.txt 2>&1; echo "hh rc=$?"; cut -c1-150 gpurun_out/bis2_hh.txt
