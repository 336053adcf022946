#!/bin/bash
# cfg3-aao launch list + full capture of its GEMMs (host sweep loop: ncu cannot profile
# kernel nodes of graphs with conditional nodes; same kernels, one graph per sweep).
export PYTHONPATH=. PE_NO_DEVICE_LOOP=1
O=gpurun_out
P="python tools/profile_step.py --workload cfg3-aao --max-iter 40"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/launches_cfg3aao.csv $P > $O/ncu_l3.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:gemm -s 30 -c 3 -f -o $O/ncu_cfg3_gemm $P > $O/ncu_g3.log 2>&1
tail -n 2 $O/ncu_l3.log; tail -n 2 $O/ncu_g3.log
