# session 2 of round 2, call a: board power under DGEMM / HBM copy / leaf kernel; GEMM engine probe 2 and 1 CTAs/SM
O=gpurun_out/${OUT:-s2a}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 300 ./tools/gemm/gemm_bench 2 > $O/gemm2.txt 2>&1
timeout 300 ./tools/gemm/gemm_bench 1 > $O/gemm1.txt 2>&1
timeout 400 python tools/probe/power_probe.py > $O/power.json 2> $O/power.err
