#!/bin/bash
# Round capture on one B200: bench lines (with CPU baselines) for every workload, the ncu
# launch list of the default bench command, and one `ncu --set full` capture of the top
# kernels of one cfg2-aao step.  Outputs under gpurun_out/; summaries go to profiles/.
set -u
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -1 gpurun_out/bench_default.json
for w in ${WORKLOADS:-cfg2-seq cfg4-seq cfg0-seq cfg1-aao}; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  tail -1 gpurun_out/bench_$w.json | cut -c1-300
done
if [ -f data/sys_cfg3.npz ] && [ -z "${NO_CFG3:-}" ]; then
  timeout 1500 python bench.py --workload cfg3-aao --steps 2 --warmup 3 > gpurun_out/bench_cfg3-aao.json 2> gpurun_out/bench_cfg3-aao.err
  tail -1 gpurun_out/bench_cfg3-aao.json | cut -c1-300
fi
# launch list of the default bench command itself (a run under ncu is never a bench value)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 \
  --launch-count 1200 --csv --log-file gpurun_out/launches_bench_cfg2aao.csv \
  python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
python tools/launch_summary.py --grid gpurun_out/launches_bench_cfg2aao.csv
# full capture: the three GEMM shapes + scans + decide of one step (profile_step range)
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  --launch-skip 12 --launch-count 6 -o gpurun_out/full_cfg2aao python tools/profile_step.py \
  --workload cfg2-aao > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
