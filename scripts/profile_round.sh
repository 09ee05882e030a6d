# ncu --set full of the K2 kernels (one launch each, second filter) and the
# launch list of the bench command; outputs under gpurun_out/
cd ${GRAFT_REPO_ROOT:-.}
for k in ${KERNELS:-qrcp qform}; do
  case $k in
    qrcp)  sel="-k regex:qrcp -s 1 -c 1" ;;
    qform) sel="-k regex:qform -s 1 -c 1" ;;
    wy64)  sel="-k regex:wy_apply -s 1 -c 1" ;;
    panel) sel="-k regex:panel -s 2 -c 1" ;;
  esac
  timeout 400 ncu --set full --clock-control none --import-source on $sel -o gpurun_out/p_$k python scripts/profile_filter.py cfg4 > gpurun_out/p_$k.log 2>&1
done
if [ -n "$LAUNCHES" ]; then
  timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/b11.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_launches.csv 2>&1
fi
ls gpurun_out
