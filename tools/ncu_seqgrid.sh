#!/bin/bash
# ncu --set full (with source) of the all-SM sequential chain kernel at cfg2-seq
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seqgrid_kernel -s 4 -c 1 -f \
    -o $O/ncu_seqgrid python tools/seq_probe.py cfg2-seq > $O/ncu_seqgrid.log 2>&1
tail -n 4 $O/ncu_seqgrid.log
ls -la $O/ncu_seqgrid.ncu-rep
