mkdir -p gpurun_out
V=paper_2502_04077_b200/lib/variants
for v in "paper_2502_04077_b200/lib/libattnpred.so" $V/s1000.so $V/s8000.so; do echo "lib=$v"; ATTNPRED_LIB=$v ATTNPRED_FUSED_SELECT=1 timeout 300 python scripts/dbg/forecast_knobs.py; ATTNPRED_LIB=$v ATTNPRED_FUSED_SELECT=1 HEADS=8 timeout 300 python scripts/wsm_cta.py 2>&1 | grep "prod_last\|exit \|roles\|group0"; done
