mkdir -p gpurun_out/wsm
timeout 240 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_gpu_trace_replay.py -x -q > gpurun_out/wsm/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/wsm/parity.log
for k in wsm ws; do
  ATTNPRED_FORECAST_KERNEL=$k timeout 60 python scripts/bench_select.py --heads 8 --steps 20 --warmup 4 > gpurun_out/wsm/sel_kv_$k.json 2>&1
  ATTNPRED_FORECAST_KERNEL=$k timeout 60 python scripts/bench_select.py --steps 20 --warmup 4 > gpurun_out/wsm/sel_head_$k.json 2>&1
done
