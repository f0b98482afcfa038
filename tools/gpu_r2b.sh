mkdir -p gpurun_out
timeout 600 python -m paper_2504_15465_b200.rightsize --quick --reps 2 > gpurun_out/rightsize.json 2> gpurun_out/rightsize.err; echo "rightsize rc=$?"; tail -3 gpurun_out/rightsize.err
python -c "
import json; d=json.load(open('gpurun_out/rightsize.json'))
for b in d['bodies']: print(b['body'], 'ref t*', b['t_star'], round(b['slowdown'],3), 'b200 t*', b['b200']['t_star'], round(b['b200']['slowdown'],3), b['b200']['probes'])
print('savings ref', d['mean_capacity_savings'], 'b200', d['b200_mean_capacity_savings'], 'max slow', d['b200_max_slowdown'])"
timeout 1200 python tools/hybrid_variants.py --horizon-ms 1000 --reps 3 2>&1 | tail -8
