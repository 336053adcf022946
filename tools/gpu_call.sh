mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_cem.py -q -p no:cacheprovider -k "rowbalanced or config4 or ensemble or cem" 2>&1 | tail -4 > gpurun_out/pytest16.log
timeout 600 python bench.py --workload cfg4-seq --steps 5 --warmup 3 --no-cpu > gpurun_out/bench16_cfg4.json 2> gpurun_out/bench16_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.min.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --profile-from-start off -k regex:rowbal --csv --log-file gpurun_out/launches16_cfg4.csv python tools/profile_step.py --workload cfg4-seq > /dev/null 2>&1
export PE_NO_GRAPHS=1
# launch list of one cfg3-aao step (time + DRAM bytes per launch; graphs off so every kernel is visible)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_cfg3.csv python tools/profile_step.py --workload cfg3-aao > gpurun_out/ncu_l3.log 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg3.csv > gpurun_out/launch_summary_cfg3.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_fast --launch-skip 4 --launch-count 1 -o gpurun_out/full_cfg3_gemm python tools/profile_step.py --workload cfg3-aao > gpurun_out/ncu_f3.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --profile-from-start off -k regex:modal_ --launch-skip 30 --launch-count 3 -o gpurun_out/full_cfg2_scans python tools/profile_step.py --workload cfg2-aao > gpurun_out/ncu_s2.log 2>&1
ls gpurun_out/*.ncu-rep
