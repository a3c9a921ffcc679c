# Round profile bundle: bench line, step launch list, ncu captures of the GEMV and sparse attention kernels.
set -u
out=gpurun_out/prof3
mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_step.csv python scripts/profile_step.py --what step > $out/l.log 2>&1
python scripts/launches.py $out/launches_step.csv > $out/launches_step.summary.txt 2>&1
timeout 300 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemv_stream \
  --launch-skip 2 -c 1 -o $out/gemv_gate_up python scripts/profile_step.py --what step > $out/g.log 2>&1
timeout 300 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:sparse_cluster \
  -c 1 -o $out/sparse python scripts/profile_step.py --what step > $out/s.log 2>&1
