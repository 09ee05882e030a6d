for L in paper_2506_17626_b200/libfeatlsq_b200.so paper_2506_17626_b200/_build/var/nomma.so paper_2506_17626_b200/_build/var/noload.so; do
FEATLSQ_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:qform -c 1 --csv python scripts/profile_filter.py cfg4 > gpurun_out/qf.csv 2>&1
echo $(basename $L) $(grep -E "gpu__time|pipe_tensor|wavefronts" gpurun_out/qf.csv | awk -F, '{printf "%s=%s ", $(NF-2), $NF}')
done
