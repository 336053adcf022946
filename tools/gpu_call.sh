mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 2>&1 | tail -30 > gpurun_out/pytest4.log
python tools/wr_stop_compare.py > gpurun_out/wr_stop_compare.log 2>&1
timeout 600 python bench.py --workload cfg2-aao --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_cfg2.json 2> gpurun_out/bench4_cfg2.err
PE_NO_DEVICE_LOOP=1 timeout 600 python bench.py --workload cfg2-aao --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_cfg2_noloop.json 2> gpurun_out/bench4_cfg2_noloop.err
tail -3 gpurun_out/pytest4.log
