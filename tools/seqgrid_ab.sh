#!/bin/bash
# A/B of seqgrid build variants (build/variants/libpe_<name>.so) at cfg2-seq
out=gpurun_out/seqgrid_ab.log
: > $out
cp paper_2411_09244_b200/libpe.so /tmp/libpe_keep.so
for v in "$@"; do
  cp build/variants/libpe_$v.so paper_2411_09244_b200/libpe.so
  echo "== $v" >> $out
  PE_SEQGRID_TRACE=1 timeout 300 python tools/seq_probe.py cfg2-seq 2>&1 | tail -3 >> $out
done
cp /tmp/libpe_keep.so paper_2411_09244_b200/libpe.so
cat $out
