mkdir -p gpurun_out
# launch list of one cfg3-aao step (time + DRAM bytes per launch)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_cfg3.csv python tools/profile_step.py --workload cfg3-aao > gpurun_out/ncu_l3.log 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg3.csv > gpurun_out/launch_summary_cfg3.txt 2>&1
# full capture of the cfg3 rhs GEMM (the dominant kernel): one launch in situ
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_fast --launch-skip 4 --launch-count 1 -o gpurun_out/full_cfg3_gemm python tools/profile_step.py --workload cfg3-aao > gpurun_out/ncu_f3.log 2>&1
# scans of cfg2-aao in situ with --cache-control none (no flush between kernels)
timeout 900 ncu --set full --cache-control none --clock-control none --profile-from-start off -k regex:modal_ --launch-skip 30 --launch-count 3 -o gpurun_out/full_cfg2_scans python tools/profile_step.py --workload cfg2-aao > gpurun_out/ncu_s2.log 2>&1
ls gpurun_out
