# Round-2 closing profile bundle: launch list of one decode step (profile_step.py, NVTX-free start/stop),
# --set full of the forecaster and of the band top-k at the bench shape.
set -u
out=gpurun_out/prof_r2
mkdir -p $out
timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_step_b1.csv python scripts/profile_step.py --what step --batch 1 > $out/l1.log 2>&1
python scripts/launches.py $out/launches_step_b1.csv > $out/launches_step_b1.summary.txt 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:conv_forecast_wsm \
  -c 1 -o $out/forecast_wsm_b1 python scripts/profile_step.py --what step --batch 1 > $out/f.log 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:sel_topk_band \
  -c 1 -o $out/topk_band_b1 python scripts/profile_step.py --what step --batch 1 > $out/t.log 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:calib_tc \
  -c 1 -o $out/calib_b1 python scripts/profile_step.py --what calib --batch 1 > $out/c.log 2>&1
ls $out
timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_calib_b1.csv python scripts/profile_step.py --what calib --batch 1 > $out/l2.log 2>&1
python scripts/launches.py $out/launches_calib_b1.csv > $out/launches_calib_b1.summary.txt 2>&1
