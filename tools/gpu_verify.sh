# Regression pass after a dispatcher change: GPU tests, configs #2/#3 as the
# bench runs them, and the split-K stress variant of config #3.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.txt)"
grep "^FAILED\|GpuosError:" gpurun_out/pytest_gpu.txt | head -5
for i in 1 2 3 4 5 6; do
  timeout 300 python tools/hybrid_variants.py --only A --reps 3 --splits 3,4,3,4 > gpurun_out/soak_$i.txt 2>&1
  echo "soak $i rc=$? $(grep -o 'GpuosError.*' gpurun_out/soak_$i.txt | cut -c1-150)"
done
timeout 900 python tools/hang_hunt2.py 2 > gpurun_out/hh.txt 2>&1; echo "hh rc=$?"; cut -c1-200 gpurun_out/hh.txt | tail -3
