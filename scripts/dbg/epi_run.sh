mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python scripts/bench_attention.py 2>&1 | tail -1 | cut -c1-120; done
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_decode.py tests/test_gpu_head_split.py -x -q 2>&1 | tail -2
