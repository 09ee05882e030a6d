# time the qrcp kernel (ncu launch durations) for library variants at given grids
for L in ${LIBS}; do
  for G in 1024; do
    FEATLSQ_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qrcp --csv python scripts/profile_filter.py cfg4 > gpurun_out/qv.csv 2>&1
    echo "$(basename $L) G=$G $(grep kept gpurun_out/qv.csv | tail -1) $(grep -E 'gpu__time|dram__bytes' gpurun_out/qv.csv | tail -3 | awk -F, '{printf "%s=%s ", $(NF-2), $NF}')"
  done
done
