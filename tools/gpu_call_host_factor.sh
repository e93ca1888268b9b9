# configs[4] solve_bvp breakdown with the device interface assembly (default) — refreshes r01_host_factor
set -x
O=gpurun_out/${OUT:-c12}; mkdir -p $O
timeout 1500 python tools/host_factor.py --ps 6,8,10,12,14,16 > $O/host_factor.jsonl 2> $O/host_factor.err
ls -la $O
