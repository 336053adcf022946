#!/bin/bash
# What the driver runs at round end, in its order, on one box: GPU tests, smoke, the
# reference arm, the default bench; then the fine-scale bench record.
O=gpurun_out/driverlike
mkdir -p $O
python -m pytest tests -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "pytest rc $?" >> $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err
python bench.py --gpus 1 > $O/bench_default_cfg3.json 2> $O/bench_default_cfg3.err
python tools/bench_finescale.py --nx 100 256 512 > $O/bench_finescale.jsonl 2>/dev/null
PE_FINE_CHAIN=1 python tools/bench_finescale.py --nx 100 >> $O/bench_finescale.jsonl 2>/dev/null
tail -n 3 $O/gpu_tests.log $O/smoke.log
cut -c1-400 $O/bench_reference_arm.json
cut -c1-300 $O/bench_default_cfg3.json
