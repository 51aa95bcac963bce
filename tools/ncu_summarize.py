"""Summarise an ncu --set full report of the conv kernel into profiles/ (tracked).

    python tools/ncu_summarize.py gpurun_out/prof_fic.ncu-rep --layers "l4.1;l1.1;l3.1" \
        --revision "..." --out profiles/ncu_summary.json

Per captured launch: duration, DRAM bytes read / written (the roofline `traffic`),
tensor-pipe activity, SM throughput, registers, grid, executed instructions.
"""
import argparse
import csv
import io
import json
import subprocess

METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "imma_subpipe_active_cycles": "TPC.TriageCompute.sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_cycles": "sm__cycles_elapsed.avg",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "warp_instructions": "smsp__inst_executed.sum",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3, "nsecond": 1e-3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--layers", default="")
    ap.add_argument("--revision", default="")
    ap.add_argument("--command", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-layer", type=int, default=1, help="index of the launch whose DRAM bytes are `traffic`")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    names = a.layers.split(";") if a.layers else []
    out = []
    for n, r in enumerate(rows[2:]):
        e = {"layer": names[n] if n < len(names) else str(n), "kernel": r[hdr.index("Kernel Name")]}
        for key, m in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = float(r[i].replace(",", "")) if r[i] and r[i] != "no data" else None
            if v is not None and units[i] in SCALE:
                v *= SCALE[units[i]]
            e[key] = v
        out.append(e)
    t = out[a.traffic_layer]
    summary = {"revision": a.revision, "command": a.command,
               "note": "ncu replays with cold caches and serialised launches: absolute times are higher than the "
                       "graph-timed bench; read shares and counters",
               "traffic_bytes_per_launch": int(t["dram_read_bytes"] + t["dram_write_bytes"]),
               "traffic_layer": t["layer"], "launches": out}
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
