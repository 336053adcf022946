#!/bin/bash
# kernel durations (ncu launch list) of seqgrid build variants at cfg2-seq
cp paper_2411_09244_b200/libpe.so /tmp/libpe_keep.so
for v in "$@"; do
  [ $v = current ] && cp /tmp/libpe_keep.so paper_2411_09244_b200/libpe.so || cp build/variants/libpe_$v.so paper_2411_09244_b200/libpe.so
  echo "== $v"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:seqgrid_kernel -s 4 -c 6 --csv python tools/seq_probe.py cfg2-seq 2>/dev/null | grep seqgrid_kernel | awk -F, '{print $NF}' | tr '\n' ' '
  echo
done
cp /tmp/libpe_keep.so paper_2411_09244_b200/libpe.so
