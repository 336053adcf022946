mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "rowbalanced or config4 or ensemble or coarse or sharded" 2>&1 | tail -15 > gpurun_out/pytest6.log
timeout 600 python bench.py --workload cfg4-seq --steps 5 --warmup 3 --no-cpu > gpurun_out/bench6_cfg4.json 2> gpurun_out/bench6_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches6_cfg4.csv python tools/profile_step.py --workload cfg4-seq > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches6_cfg4.csv > gpurun_out/launch6_cfg4.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --launch-skip 2 --launch-count 1 -o gpurun_out/full6_cfg4 python tools/profile_step.py --workload cfg4-seq > gpurun_out/ncu6.log 2>&1
tail -3 gpurun_out/pytest6.log
