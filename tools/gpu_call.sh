mkdir -p gpurun_out
for v in old pf2; do ./build/probe/p_$v 64 600 32; ./build/probe/p_$v 1 8192 16; ./build/probe/p_$v 8 4096 16; ./build/probe/p_$v 2 1201 8; done > gpurun_out/probe23.txt 2>&1
timeout 600 python bench.py --workload cfg4-seq --steps 5 --warmup 3 --no-cpu > gpurun_out/bench23_cfg4.json 2> gpurun_out/bench23_cfg4.err
