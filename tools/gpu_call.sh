mkdir -p gpurun_out
python -m pytest tests/test_gpu_cem.py -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest14.log
timeout 900 python tools/cem_build_bench.py cfg2 > gpurun_out/cem_cfg2.log 2>&1
timeout 1500 python tools/cem_build_bench.py cfg3 > gpurun_out/cem_cfg3.log 2>&1
tail -3 gpurun_out/pytest14.log
