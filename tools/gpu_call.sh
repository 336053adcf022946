set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_reference_api.py -q -p no:cacheprovider -k example1 2>&1 | grep -E "assert|Error|counts|passed|failed" | head -20 > gpurun_out/ex1.log
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "baseline_config2" 2>&1 | tail -15 > gpurun_out/cfg2test.log
python tools/wr_stop_compare.py > gpurun_out/wr_stop_compare.log 2>&1
# launch lists of one step of the sequential workloads
for w in cfg4-seq cfg2-seq; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$w.csv python tools/profile_step.py --workload $w > gpurun_out/ncu_l_$w.log 2>&1
done
python tools/launch_summary.py gpurun_out/launches_cfg4-seq.csv > gpurun_out/launch_summary_cfg4.txt 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg2-seq.csv > gpurun_out/launch_summary_cfg2seq.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --launch-skip 2 --launch-count 2 -o gpurun_out/full_cfg4seq python tools/profile_step.py --workload cfg4-seq > gpurun_out/ncu_full_cfg4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --launch-count 3 -o gpurun_out/full_cfg2seq python tools/profile_step.py --workload cfg2-seq > gpurun_out/ncu_full_cfg2seq.log 2>&1
ls -la gpurun_out
