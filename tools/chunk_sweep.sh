# Member-chunk size of the sequential ensemble sweep (PE_SEQ_CHUNK), in situ via bench.py.
for c in 64 32 22 16; do
  PE_SEQ_CHUNK=$c timeout 300 python bench.py --workload cfg4-seq --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunk $c', d['ms_per_step'], d['value'])"
done
