mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "rowbalanced or config4" 2>&1 | tail -3 > gpurun_out/pytest10.log
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.min.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --profile-from-start off -k regex:rowbal --csv --log-file gpurun_out/launches10_cfg4.csv python tools/profile_step.py --workload cfg4-seq > /dev/null 2>&1
timeout 600 python bench.py --workload cfg4-seq --steps 5 --warmup 3 --no-cpu > gpurun_out/bench10_cfg4.json 2> gpurun_out/bench10_cfg4.err
