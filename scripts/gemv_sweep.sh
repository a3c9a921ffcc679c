mkdir -p gpurun_out/gsweep9
for cfg in "4096 8" "4096 2" "2048 3" "2048 4" "1024 6"; do
 set -- $cfg
 ATTNPRED_GEMV_SLAB=$1 ATTNPRED_GEMV_STAGES=$2 timeout 120 python scripts/bench_gemv.py --rows 1 > gpurun_out/gsweep9/s$1_n$2.json 2>&1
 ATTNPRED_GEMV_SLAB=$1 ATTNPRED_GEMV_STAGES=$2 timeout 600 python bench.py --no-alt --no-dense --steps 20 > gpurun_out/gsweep9/bench_s$1_n$2.json 2> /dev/null
done
