# call c: GEMM probe ring depth (3/4/5 stages) with 1 and 2 CTAs per SM, and one active warp per SMSP at 4 stages
O=gpurun_out/${OUT:-s2c}; mkdir -p $O
for v in s4 s5 s4idle; do for c in 1 2; do timeout 300 ./tools/gemm/gemm_bench_$v $c > $O/gemm_${v}_$c.txt 2>&1; done; done
