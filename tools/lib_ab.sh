#!/bin/bash
# A/B of whole-library builds (build/variants/libpe_<name>.so, or "current") on a bench workload
wl=$1; shift
cp paper_2411_09244_b200/libpe.so /tmp/libpe_keep.so
for v in "$@"; do
  [ $v = current ] && cp /tmp/libpe_keep.so paper_2411_09244_b200/libpe.so || cp build/variants/libpe_$v.so paper_2411_09244_b200/libpe.so
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', j['ms_per_step'], j['roofline']['frac'], j['roofline']['gemm_ms'], j['roofline'].get('other_kernels_ms'))"
done
cp /tmp/libpe_keep.so paper_2411_09244_b200/libpe.so
