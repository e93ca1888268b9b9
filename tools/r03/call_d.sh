# call d: GEMM probe mainloop variants (fragment double buffer, non-volatile DMMA asm, 255-register bound), 1/2 CTAs, 1 warp per SMSP
O=gpurun_out/${OUT:-s2d}; mkdir -p $O
for v in base fp nv fpnv fpidle fpnvidle lb1 lb1idle; do for c in 1 2; do timeout 300 ./tools/gemm/gemm_bench_$v $c > $O/gemm_${v}_$c.txt 2>&1; done; done
