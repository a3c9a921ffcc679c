mkdir -p gpurun_out/ts
rm -f gpurun_out/ts/dbg.txt
for d in 0 1 2 4 3 5 6 7; do
  echo "dbg=$d $(ATTNPRED_FORECAST_DEBUG=$d timeout 60 python scripts/bench_select.py --heads 8 --steps 20 --warmup 4 2>&1 | grep -o '"us_per_step_median": [0-9.]*')" >> gpurun_out/ts/dbg.txt
done
