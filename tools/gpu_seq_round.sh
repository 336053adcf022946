#!/bin/bash
# cfg2-seq after the seqgrid change: full GPU suite, bench line, ncu capture, launch list
O=gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gpu_tests_seq.log 2>&1; tail -3 $O/gpu_tests_seq.log
timeout 600 python bench.py --workload cfg2-seq --steps 20 --warmup 5 > $O/bench_cfg2-seq.json 2> $O/bench_cfg2-seq.err; tail -c 600 $O/bench_cfg2-seq.json
timeout 600 python bench.py --workload cfg4-seq --steps 10 --warmup 3 --no-cpu > $O/bench_cfg4-seq.json 2> $O/bench_cfg4-seq.err; tail -c 300 $O/bench_cfg4-seq.json
bash tools/ncu_seqgrid.sh
