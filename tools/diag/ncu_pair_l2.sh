set -x
M="dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum"
export N=32768 FLAGS=0
for cfg in "1 1" "1 0" "0 1" "0 0"; do set -- $cfg
  GMP_TC2_RASTER=$1 GMP_TC2_HINTS=$2 ncu --metrics $M --clock-control none -k regex:k_tc2_class --csv python tools/diag/pair_vs_cublas.py > gpurun_out/ncu_pair_r$1h$2.csv 2>/dev/null
done
