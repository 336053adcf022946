# Time every cp.async tile variant on the cfg4 ensemble step shape (PE_GEMM_VARIANT forces one).
for v in -1 0 1 2 3 5 6 7 8 9 10 11 12 13 14 15 16 17 18 19; do
  if [ $v -ge 0 ]; then export PE_GEMM_VARIANT=$v; else unset PE_GEMM_VARIANT; fi
  echo "variant $v"; PE_GEMM_TRACE=1 GEMM_BENCH_ONLY="cfg4 seq step chunk" timeout 120 python tools/gemm_bench.py 2>&1 | grep -E "cfg4|variant=" | sort -u | head -3
done
