mkdir -p gpurun_out/gsweep8
timeout 300 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_decode.py -x -q > gpurun_out/gsweep8/tests.log 2>&1
timeout 120 python scripts/bench_gemv.py --rows 1 > gpurun_out/gsweep8/ns1.json 2>&1
timeout 120 python scripts/bench_gemv.py --rows 1 --ns 4 > gpurun_out/gsweep8/ns4.json 2>&1
timeout 600 python bench.py --no-alt > gpurun_out/gsweep8/bench.json 2> gpurun_out/gsweep8/bench.err
