"""Distil an ncu --set full capture of one featurize launch into
profiles/featurize_ncu.json: DRAM bytes per prompt (bench.py scales it to its
own launch for roofline.traffic) and the pipe utilisations behind the
issue-bound claim. Usage: python tools/ncu_to_json.py rep.ncu-rep n_prompts out.json"""
import csv
import io
import json
import subprocess
import sys

rep, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else "one launch over the first n prompts of the C4 workload"
raw = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
h, units, v = raw[0], raw[1], raw[2]
d = dict(zip(h, v))
u = dict(zip(h, units))


def num(k):
    x = float(d[k].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}.get(u.get(k, ""), 1)
    return x * scale


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
j = {
    "kernel": d.get("Kernel Name", ""),
    "prompts": n,
    "dram_read_bytes": rd,
    "dram_write_bytes": wr,
    "dram_bytes_per_prompt": (rd + wr) / n,
    "duration_ns": num("gpu__time_duration.sum"),
    "alu_pipe_pct_active": float(d["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]),
    "fma_pipe_pct_active": float(d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]),
    "lsu_wavefronts_pct": float(d["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]),
    "issue_active_pct": float(d["sm__inst_issued.avg.pct_of_peak_sustained_active"]),
    "ipc_active": float(d["sm__inst_executed.avg.per_cycle_active"]),
    "warp_instructions": num("smsp__inst_executed.sum"),
    "fp64_pipe_pct_active": float(d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "nan")),
    "dram_throughput_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
    "note": "ncu --set full --clock-control none, " + note,
}
json.dump(j, open(out, "w"), indent=1)
print(json.dumps(j, indent=1))
