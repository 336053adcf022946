#!/bin/bash
# One GPU pass: tests + bench lines for the main workloads (+ optional launch list)
set -u
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for w in ${WORKLOADS:-cfg2-aao cfg2-seq cfg0-seq cfg1-aao}; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 ${BENCH_ARGS:---no-cpu} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w value %.4g ms/step %.4g roof %.3f achieved %.2f share %.2f e2e %.4g launches %d' % (d['value'], d['ms_per_step'], r['frac'], r['achieved'], r['gemm_share_of_step'], d['e2e']['value'], d['gpu_launches']))" || tail -3 gpurun_out/bench_$w.err
done
if [ -n "${PROFILE:-}" ]; then
  timeout 300 python tools/profile_step.py --workload $PROFILE > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_$PROFILE.csv python tools/profile_step.py --workload $PROFILE > gpurun_out/ncu1.log 2>&1
  python tools/launch_summary.py --grid gpurun_out/launches_$PROFILE.csv
fi
