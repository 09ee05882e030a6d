# Round-2 evidence (one GPU): ncu --set full of the new K1 and of K2b,
# K1's FP64 op counts and DRAM bytes, and the launch list of the bench
# command; outputs under gpurun_out/. Each ncu run only after its command
# exited 0 without ncu.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python scripts/profile_assemble.py cfg4 > gpurun_out/p2_asm_plain.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:assemble_kernel -s 1 -c 1 \
    -o gpurun_out/p2_asm python scripts/profile_assemble.py cfg4 > gpurun_out/p2_asm.log 2>&1 && \
  timeout 300 ncu --clock-control none -k regex:assemble_kernel -s 1 -c 1 --csv --metrics \
    smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum \
    python scripts/profile_assemble.py cfg4 > gpurun_out/p2_asm_flops.csv 2>&1
python scripts/profile_filter.py cfg4 > gpurun_out/p2_filter_plain.log 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:qrcp -s 1 -c 1 \
    -o gpurun_out/p2_qrcp python scripts/profile_filter.py cfg4 > gpurun_out/p2_qrcp.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-configs --no-paper > gpurun_out/p2_bench_plain.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-configs --no-paper > gpurun_out/p2_bench_launches.csv 2>&1
ls gpurun_out | grep p2_
