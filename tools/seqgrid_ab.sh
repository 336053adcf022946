#!/bin/bash
# A/B of seqgrid build variants (build/variants/libpe_<name>.so) at cfg2-seq: in-kernel trace
# (PE_SEQGRID_TRACE adds a malloc / sync / free per call, so its event times are not
# comparable) and an untraced event-timed run
out=gpurun_out/seqgrid_ab.log
: > $out
cp paper_2411_09244_b200/libpe.so /tmp/libpe_keep.so
for v in "$@"; do
  [ $v = current ] && cp /tmp/libpe_keep.so paper_2411_09244_b200/libpe.so || cp build/variants/libpe_$v.so paper_2411_09244_b200/libpe.so
  echo "== $v" >> $out
  PE_SEQGRID_TRACE=1 timeout 300 python tools/seq_probe.py cfg2-seq 2>&1 | grep "seqgrid" | tail -2 >> $out
  timeout 300 python tools/seq_probe.py cfg2-seq 2>&1 | tail -2 >> $out
done
cp /tmp/libpe_keep.so paper_2411_09244_b200/libpe.so
cat $out
