mkdir -p gpurun_out/ts
ATTNPRED_FORECAST_KERNEL=ts timeout 240 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ts/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/ts/parity.log
ATTNPRED_FORECAST_KERNEL=ts timeout 60 python scripts/bench_select.py --heads 8 --steps 20 --warmup 4 > gpurun_out/ts/sel_kv.json 2>&1
ATTNPRED_FORECAST_KERNEL=ws timeout 60 python scripts/bench_select.py --heads 8 --steps 20 --warmup 4 > gpurun_out/ts/sel_kv_ws.json 2>&1
timeout 60 python scripts/bench_select.py --steps 20 --warmup 4 > gpurun_out/ts/sel_head.json 2>&1
timeout 60 python scripts/ws_trace.py > gpurun_out/ts/trace.txt 2>&1
