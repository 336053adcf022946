#!/bin/bash
# seqgrid plan sweep at cfg2-seq: chain-group width (ct) x groups per CTA (H)
out=gpurun_out/seqgrid_sweep.log
: > $out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -m gpu -k "seq or chain" 2>&1 | tail -5 >> $out
for cfg in ${SWEEP:-"16 1" "8 2" "16 2" "8 4" "0 0"}; do
  set -- $cfg
  echo "== ct=$1 H=$2" >> $out
  PE_SEQGRID_CT=$1 PE_SEQGRID_H=$2 PE_SEQGRID_TRACE=1 timeout 300 python tools/seq_probe.py cfg2-seq 2>&1 | tail -3 >> $out
done
