# Second profile bundle of round 1: GPU tests, smoke, bench lines (batch 1 headline, batch 8 = cfg5 per-GPU
# share), ncu launch lists of one decode step at batch 1 / 8, and --set full captures of the batch-8 kernels.
set -u
out=gpurun_out/prof4
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 900 python bench.py --batch 8 --steps 20 --warmup 3 > $out/bench_b8.json 2> $out/bench_b8.err
for b in 1 8; do
  timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/launches_step_b$b.csv python scripts/profile_step.py --what step --batch $b > $out/l$b.log 2>&1
  python scripts/launches.py $out/launches_step_b$b.csv > $out/launches_step_b$b.summary.txt 2>&1
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file $out/launches_bench_steps.csv python bench.py --steps 2 --warmup 3 --no-alt --no-dense > $out/lb.log 2>&1
python scripts/launches.py $out/launches_bench_steps.csv > $out/launches_bench_steps.summary.txt 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_tc \
  --launch-skip 2 -c 1 -o $out/gemm_tc_gate_up_b8 python scripts/profile_step.py --what step --batch 8 > $out/g.log 2>&1
timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:sparse_cluster \
  -c 1 -o $out/sparse_b8 python scripts/profile_step.py --what step --batch 8 > $out/s.log 2>&1
ls $out
