M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active
CFG=3 timeout 600 ncu --metrics $M --clock-control none -k regex:'k_gs|k_mul_scaled|k_lincomb|k_cg_' --launch-skip 300 -c 60 --csv --log-file gpurun_out/ncu_gs.csv python tools/step_timing.py > gpurun_out/ncu_gs.log 2>&1
