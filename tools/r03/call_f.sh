O=gpurun_out/${OUT:-s2f}; mkdir -p $O
for v in l2 l2idle l2s4idle; do for c in 1 2; do timeout 300 ./tools/gemm/gemm_bench_$v $c > $O/gemm_${v}_$c.txt 2>&1; done; done
