set -x
cd $GRAFT_REPO_ROOT
timeout 400 ncu --set full --clock-control none --import-source on -k regex:qrcp -s 1 -c 1 -o gpurun_out/p_qrcp python scripts/profile_filter.py cfg4 > gpurun_out/p1.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:qform -s 1 -c 1 -o gpurun_out/p_qform python scripts/profile_filter.py cfg4 > gpurun_out/p2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wy_apply -s 1 -c 1 -o gpurun_out/p_wy64 python scripts/profile_filter.py cfg4 > gpurun_out/p3.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:panel -s 2 -c 1 -o gpurun_out/p_panel python scripts/profile_filter.py cfg4 > gpurun_out/p4.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/b11.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_launches.csv 2>&1
ls -la gpurun_out
