# Round-2 (third session) evidence, one GPU: ncu --set full of the reworked
# panel kernel and of K2b, and the launch list of the bench command; outputs
# under gpurun_out/. Each ncu run only after its command exited 0 without ncu.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python scripts/profile_filter.py cfg4 > gpurun_out/p3_filter_plain.log 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 18 -c 1 \
    -o gpurun_out/p3_panel python scripts/profile_filter.py cfg4 > gpurun_out/p3_panel.log 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:qrcp -s 1 -c 1 \
    -o gpurun_out/p3_qrcp python scripts/profile_filter.py cfg4 > gpurun_out/p3_qrcp.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-configs --no-paper > gpurun_out/p3_bench_plain.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-configs --no-paper > gpurun_out/p3_bench_launches.csv 2>&1
ls -la gpurun_out | grep p3_
