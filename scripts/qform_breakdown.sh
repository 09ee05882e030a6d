# qform timing-experiment variants (QF_NO_LOAD / QF_NO_SYNC / QF_NO_MMA builds)
for L in ${LIBS}; do
FEATLSQ_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:qform -c 1 --csv python scripts/profile_filter.py cfg4 > gpurun_out/qf.csv 2>&1
echo $(basename $L) $(grep -E "gpu__time|pipe_tensor" gpurun_out/qf.csv | awk -F, '{printf "%s=%s ", $(NF-2), $NF}')
done
