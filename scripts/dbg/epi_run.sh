mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_decode.py tests/test_gpu_head_split.py tests/test_gpu_prefetch.py -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_calib2.json 2> gpurun_out/bench_calib2.err; tail -c 200 gpurun_out/bench_calib2.json
