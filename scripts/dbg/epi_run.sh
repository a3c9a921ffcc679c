mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/bench_attention.py 2>&1 | tail -1 | cut -c1-200
ATTNPRED_LIB=paper_2502_04077_b200/lib/variants/att_trace.so timeout 300 python scripts/bench_attention.py 2>&1 | tail -1 | cut -c1-200
done
timeout 300 python scripts/attn_trace.py 2>&1 | tail -10
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_decode.py -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_notrace.json 2> gpurun_out/bench_notrace.err; tail -c 150 gpurun_out/bench_notrace.json
