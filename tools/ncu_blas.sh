set -x
CFG=3 python tools/step_timing.py > gpurun_out/st.log 2>&1 || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CFG=3 timeout 600 ncu --metrics $M --clock-control none -k regex:'k_mgs_part_dev|k_mul|k_lincomb|k_momentum_rhs|k_gradient|k_momentum_axis|k_momentum_diag|k_dot_part|k_sum_parts|k_scale_copy' -c 80 --csv --log-file gpurun_out/ncu_blas1.csv python tools/step_timing.py > gpurun_out/ncu1.log 2>&1
CFG=3 timeout 600 ncu --metrics $M --clock-control none -k regex:'k_cg|k_sip_axis' --launch-skip 200 -c 40 --csv --log-file gpurun_out/ncu_blas2.csv python tools/step_timing.py > gpurun_out/ncu2.log 2>&1
