# Live (ring-fed) dispatcher under ncu + the fig7 time breakdown + racecheck.
mkdir -p gpurun_out
timeout 600 python tools/fig7_breakdown.py --out gpurun_out/fig7_breakdown.json > gpurun_out/fig7_breakdown.txt 2>&1; echo "breakdown rc=$?"; tail -40 gpurun_out/fig7_breakdown.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg --clock-control none -k regex:k_worker --csv --log-file gpurun_out/ncu_fig7_live.csv python tools/fig7_breakdown.py --runs 2 > gpurun_out/ncu_fig7_live.txt 2>&1; echo "ncu live rc=$?"; tail -5 gpurun_out/ncu_fig7_live.txt; grep k_worker gpurun_out/ncu_fig7_live.csv | head
export GPUOS_PIPELINE_TIMEOUT_MS=600000
timeout 900 compute-sanitizer --tool racecheck --kernel-name kns=k_worker --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/sanitizer_racecheck.txt
