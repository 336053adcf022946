mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches9_cfg4.csv python tools/profile_step.py --workload cfg4-seq > /dev/null 2>&1
timeout 600 python bench.py --workload cfg4-seq --steps 5 --warmup 3 --no-cpu > gpurun_out/bench9_cfg4.json 2> gpurun_out/bench9_cfg4.err
