# K2b concurrency probe: qrcp kernel time on cfg4 at several persistent grid sizes
for G in ${GRIDS:-1024 296 148 74 37}; do
  FEATLSQ_QRCP_GRID=$G timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:qrcp --csv python scripts/profile_filter.py cfg4 > gpurun_out/qrcp_grid_$G.csv 2>&1
done
