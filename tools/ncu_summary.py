"""Summarise an `ncu --set full` capture of hps_leaf_kernel into profiles/<name>.json.

    python tools/ncu_summary.py gpurun_out/r2l/full16.ncu-rep --p 16 --leaves 296 \
        --capture "<command line>" --out profiles/r02_ncu_summary_p16.json

Reads the raw page (`ncu -i ... --page raw --csv`, units as ncu prints them: GB,
ms, %), takes the first hps_leaf_kernel launch in the report, and writes the
per-leaf DRAM traffic the bench's roofline `traffic` field uses.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--p", type=int, required=True)
ap.add_argument("--leaves", type=int, required=True)
ap.add_argument("--capture", default="")
ap.add_argument("--kernel-version", default="")
ap.add_argument("--out", required=True)
a = ap.parse_args()

raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
launch = next(r for r in rows[2:] if "hps_leaf_kernel" in ",".join(r))
m = dict(zip(hdr, launch))
u = dict(zip(hdr, units))


def val(name, scale_to=None):
    v = float(m[name].replace(",", ""))
    unit = u.get(name, "")
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
            "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "second": 1.0,
            "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}.get(unit, 1.0)
    return v * mult


from paper_2503_04033_b200.engine import dtn_flops_executed  # noqa: E402
q = a.p - 2
n, mb = q ** 3, 6 * q ** 2
t = val("gpu__time_duration.sum")
rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
fp64_ops = float(m["sm__ops_path_tensor_src_fp64.avg"]) * 148
out = {
    "capture": a.capture,
    "kernel_version": a.kernel_version,
    "p": a.p,
    "leaves_per_launch": a.leaves,
    "gpu_time_ms": t * 1e3,
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "traffic_bytes_per_leaf": (rd + wr) / a.leaves,
    "algorithmic_bytes_per_leaf": 8 * (4 * n + mb * mb),
    "dram_throughput_gbs": (rd + wr) / t / 1e9,
    "l2_sector_hit_rate_pct": float(m["lts__t_sector_hit_rate.pct"]),
    "dmma_pipe_active_pct": float(m["sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"]),
    "tensor_fp64_ops_per_leaf": fp64_ops / a.leaves,
    "model_executed_flops_per_leaf": dtn_flops_executed(n, mb, q),
    "registers_per_thread": int(float(m["launch__registers_per_thread"])),
    "occupancy_limit_ctas_per_sm": float(m.get("launch__occupancy_limit_registers", "nan")),
}
out["flop_per_dram_byte"] = out["tensor_fp64_ops_per_leaf"] / out["traffic_bytes_per_leaf"]
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps(out, indent=1))
