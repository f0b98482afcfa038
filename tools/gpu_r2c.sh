for b in 64 256; do for q in 37 74; do
timeout 600 python tools/train_breakdown.py --batch $b --quota $q --horizon-ms 800 2>&1 | tail -40
done; done
