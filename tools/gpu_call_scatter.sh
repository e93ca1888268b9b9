set -x
O=gpurun_out/c9; mkdir -p $O
timeout 300 python tools/scatter_bench.py --p 16 --g 6 > $O/scatter_p16.json 2> $O/scatter_p16.err
timeout 300 python tools/scatter_bench.py --p 8 --g 12 > $O/scatter_p8.json 2> $O/scatter_p8.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hps_interface_scatter -s 3 -c 1 -o $O/scatter_full python tools/scatter_bench.py --p 16 --g 6 --iters 1 > $O/ncu.log 2>&1
ls -la $O
