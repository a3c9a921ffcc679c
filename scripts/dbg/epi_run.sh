mkdir -p gpurun_out
for i in 1 2; do
ATTNPRED_FUSED_SELECT=0 timeout 300 python scripts/dbg/forecast_knobs.py
ATTNPRED_TOPK_KERNEL=radix ATTNPRED_FUSED_SELECT=0 timeout 300 python scripts/dbg/forecast_knobs.py
done
ATTNPRED_FUSED_SELECT=0 timeout 300 python scripts/dbg/sel_timing.py 2>&1 | tail -7 | head -5
ATTNPRED_TOPK_KERNEL=radix ATTNPRED_FUSED_SELECT=0 timeout 300 python scripts/dbg/sel_timing.py 2>&1 | tail -7 | head -5
ATTNPRED_FUSED_SELECT=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sel_topk_band -s 5 -c 1 -f -o gpurun_out/topk_band2 python scripts/dbg/forecast_knobs.py > gpurun_out/topk_band_ncu2.log 2>&1
