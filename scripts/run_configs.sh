#!/usr/bin/env bash
# BASELINE.json configs beyond the headline (configs[1]): one bench line each into gpurun_out/configs/.
#   cfg1: 32 heads x 4K x 64 steps of the reference's synthetic maps -> predict + top-k us/layer
#   cfg3: LongChat-7B-v1.5-32K shape, 16K ctx, budgets 256..2048 (periodic calibration, M=5)
#   cfg4: LLaMA-3.1-8B 128K with V offloaded to pinned host memory + cross-token prefetch
#         (+ resident sparse / dense comparators, prefetch GB/s, the cross-token latency model)
#   cfg5: batched decode, 8 sequences per GPU at 32K (the per-GPU share of 64 sequences on 8 GPUs)
set -u
out=gpurun_out/configs
mkdir -p "$out"
timeout 600 python bench.py --workload cfg1 --warmup 4 > "$out/cfg1_4k.json" 2> "$out/cfg1_4k.err"
for b in 256 512 1024 2048; do
  timeout 900 python bench.py --model longchat-7b-v1.5-32k --ctx 16384 --budget "$b" --no-alt --steps 20 --warmup 3 \
    --cpu-sample 4 > "$out/cfg3_longchat_16k_b$b.json" 2> "$out/cfg3_longchat_16k_b$b.err"
done
timeout 1800 python bench.py --ctx 131072 --offload --steps 20 --warmup 3 --no-alt --cpu-sample 2 \
  > "$out/cfg4_offload_128k.json" 2> "$out/cfg4_offload_128k.err"
timeout 1200 python bench.py --total-seqs 8 --steps 20 --warmup 3 --no-alt --cpu-sample 4 \
  > "$out/cfg5_8seq_32k.json" 2> "$out/cfg5_8seq_32k.err"
