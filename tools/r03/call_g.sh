O=gpurun_out/${OUT:-s2g}; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_probe -s 1 -c 1 -o $O/idle1 ./tools/gemm/gemm_bench_idle_hi 1 > $O/idle1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_probe -s 1 -c 1 -o $O/full2 ./tools/gemm/gemm_bench 2 > $O/full2.log 2>&1
ls -la $O
