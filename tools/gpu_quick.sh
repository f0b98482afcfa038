mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "dispatcher or chain" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.txt
for v in "--quantum-us 25" "--quantum-us 25 --no-lookahead" "--quantum-us 50" "--quantum-us 0"; do
n=$(echo $v | tr -d ' -')
timeout 600 python tools/fig7_breakdown.py $v --out gpurun_out/fig7_bd_$n.json > gpurun_out/fig7_bd_$n.txt 2>&1; echo "breakdown $v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/fig7_bd_$n.json')); print({k: d[k] for k in ['roofline_frac','avg_running_workers','gbs_per_running_worker','tpc_busy_frac_sampled','be_device_held_tpc_frac','lc_p99_ms']})"
done
