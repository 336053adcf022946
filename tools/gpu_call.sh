mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 2>&1 | tail -30 > gpurun_out/pytest11.log
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench11_default.json 2> gpurun_out/bench11_default.err
tail -3 gpurun_out/pytest11.log
