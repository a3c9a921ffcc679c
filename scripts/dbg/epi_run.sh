mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_32k.py tests/test_gpu_parity.py tests/test_gpu_budget.py tests/test_gpu_trace_replay.py -x -q 2>&1 | tail -1
for i in 1 2; do
timeout 300 python scripts/dbg/sel_timing.py 2>&1 | tail -7 | sed -n 3p
ATTNPRED_LIB=paper_2502_04077_b200/lib/variants/old_calib.so timeout 300 python scripts/dbg/sel_timing.py 2>&1 | tail -7 | sed -n 3p
done
timeout 600 python scripts/step_timeline.py --out gpurun_out/tl_det.json 2>&1 | grep "topk\|refine\|wall"
