cd ${GRAFT_REPO_ROOT:-.}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 6 -c 1 -o gpurun_out/p_fused python scripts/time_stages.py cfg4 10 > gpurun_out/p_fused.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/b11.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_launches.csv 2>&1
ls gpurun_out
