# per-kernel device time of one filter for library variants (ncu launch list)
for L in ${LIBS}; do
  FEATLSQ_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/profile_filter.py ${CFG:-cfg4} > gpurun_out/vl.csv 2>&1
  echo "== $(basename $L) $(grep kept gpurun_out/vl.csv | tail -1)"
  python scripts/launch_summary.py gpurun_out/vl.csv | head -${TOP:-7}
done
