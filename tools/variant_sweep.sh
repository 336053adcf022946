# Time every cp.async tile variant on the cfg2 modal shapes (PE_GEMM_VARIANT forces one).
for v in -1 0 1 5 6 11 14 15 17 18 19; do
  if [ $v -ge 0 ]; then export PE_GEMM_VARIANT=$v; else unset PE_GEMM_VARIANT; fi
  echo "variant $v"; GEMM_BENCH_ONLY=cfg2 timeout 120 python tools/gemm_bench.py 2>&1 | grep -E "rhs/g|norms"
done
