# TMA tile variant (PE_TMA_VARIANT) for the cfg4 ensemble step, in situ via bench.py.
for v in -1 6 9 10; do
  if [ $v -ge 0 ]; then export PE_TMA_VARIANT=$v; else unset PE_TMA_VARIANT; fi
  timeout 300 python bench.py --workload cfg4-seq --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('tma variant $v', d['ms_per_step'], r['gemm_ms'], r['frac'])"
done
