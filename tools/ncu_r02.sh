#!/bin/bash
# Round-2 ncu evidence: cfg3-aao launch list + full captures of its GEMMs; cfg2-aao scans
# in situ with --cache-control none (L2 write-backs of earlier kernels not billed).
set -x
export PYTHONPATH=.
# ncu cannot profile kernel nodes of graphs with conditional nodes: the host sweep loop
# launches the same kernels (one graph per sweep)
export PE_NO_DEVICE_LOOP=1
O=gpurun_out
P="python tools/profile_step.py --workload cfg3-aao --max-iter 40"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/launches_cfg3aao.csv $P > $O/ncu_l3.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:gemm -s 30 -c 3 -f -o $O/ncu_cfg3_gemm $P > $O/ncu_g3.log 2>&1
P2="python tools/profile_step.py --workload cfg2-aao --max-iter 40"
ncu --set full --clock-control none --cache-control none --import-source on --profile-from-start off \
    -k regex:modal_.scan -s 20 -c 2 -f -o $O/ncu_cfg2_scans $P2 > $O/ncu_s2.log 2>&1
for f in $O/ncu_l3.log $O/ncu_g3.log $O/ncu_s2.log; do tail -n 3 $f; done
ls -la $O
