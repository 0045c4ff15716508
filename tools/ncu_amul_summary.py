"""Summarise an ncu --set full capture of the a3 block multiply (dgemm_kp_kernel<..., 1>) into
profiles/ncu_amul_r01.json: duration, DRAM bytes per launch (read + write), tensor-pipe utilisation.
Usage: python tools/ncu_amul_summary.py gpurun_out/amul.ncu-rep profiles/ncu_amul_r01.json"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


def num(k):
    v = d.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def scaled(k):
    v = num(k)
    if v is None:
        return None
    unit = u.get(k, "")
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
                "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(unit, 1.0)


rd, wr = scaled("dram__bytes_read.sum"), scaled("dram__bytes_write.sum")
dur = scaled("gpu__time_duration.sum")
res = {"duration_unit": u.get("gpu__time_duration.sum"), "kernel": d.get("Kernel Name"), "grid": d.get("Grid Size"), "block": d.get("Block Size"),
       "duration_s": dur, "dram_bytes_read": rd, "dram_bytes_write": wr,
       "dram_bytes_per_launch": (rd or 0) + (wr or 0),
       "tensor_dp_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") or
       num("sm__inst_executed_pipe_tensor_op_dmma.avg.pct_of_peak_sustained_active"),
       "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
       "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
       "achieved_occupancy_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
       "registers": num("launch__registers_per_thread"), "source": rep}
pipes = {k: num(k) for k in hdr if "pipe_tensor" in k and k.endswith("pct_of_peak_sustained_active")}
res["tensor_pipes_pct"] = {k: v for k, v in pipes.items() if v}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
