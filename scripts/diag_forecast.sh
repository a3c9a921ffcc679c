set -u
mkdir -p gpurun_out/diag
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/tc_micro.cu -o /tmp/tc_micro && /tmp/tc_micro > gpurun_out/diag/tc_micro.txt 2>&1
for d in 0 1 2 4 3 5 6 7; do
  echo "dbg=$d" >> gpurun_out/diag/dbg.txt
  ATTNPRED_FORECAST_DEBUG=$d timeout 120 python scripts/bench_select.py --heads 8 --steps 20 --warmup 4 >> gpurun_out/diag/dbg.txt 2>&1
done
timeout 200 python scripts/ws_prof.py 8 > gpurun_out/diag/wsprof_1024.txt 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag/launches_step.csv python scripts/profile_step.py --what step > gpurun_out/diag/ncu_step.log 2>&1
python scripts/launches.py gpurun_out/diag/launches_step.csv > gpurun_out/diag/launches_step.summary.txt 2>&1
