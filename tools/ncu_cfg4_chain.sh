#!/bin/bash
# cfg4-seq after the chained row-balanced kernel and the member-cluster coarse sweep:
# bench line, launch list of one iteration, ncu --set full of the chain kernel
O=gpurun_out
timeout 600 python bench.py --workload cfg4-seq --steps 10 --warmup 3 > $O/bench_cfg4-seq.json 2> $O/bench_cfg4-seq.err; tail -c 400 $O/bench_cfg4-seq.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/launches_cfg4-seq.csv python tools/profile_cfg4.py > $O/ncu_l4.log 2>&1; tail -2 $O/ncu_l4.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:rowbal_chain -c 1 -f -o $O/ncu_rowbal_chain python tools/profile_cfg4.py > $O/ncu_g4.log 2>&1; tail -2 $O/ncu_g4.log
