# Third profile bundle of round 1 (after the conflict-free conv1 tile layout): GPU tests, bench line,
# launch list of the bench's timed steps, --set full of the forecaster at the bench shape.
set -u
out=gpurun_out/prof5
mkdir -p $out
timeout 600 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file $out/launches_bench_steps.csv python bench.py --steps 2 --warmup 3 --no-alt --no-dense > $out/lb.log 2>&1
python scripts/launches.py $out/launches_bench_steps.csv > $out/launches_bench_steps.summary.txt 2>&1
timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_step_b1.csv python scripts/profile_step.py --what step --batch 1 > $out/l1.log 2>&1
python scripts/launches.py $out/launches_step_b1.csv > $out/launches_step_b1.summary.txt 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:conv_forecast_wsm \
  -c 1 -o $out/forecast_wsm_b1 python scripts/profile_step.py --what step --batch 1 > $out/f.log 2>&1
ls $out
