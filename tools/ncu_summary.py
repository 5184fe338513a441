"""Summarise ncu output brought back in gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py --rep gpurun_out/prof_r1a.ncu-rep --launches gpurun_out/launches_r1a.csv \
        --tag r01a --config llama8b

Writes profiles/ncu_<tag>.md (per-kernel key metrics of the --set full capture and the launch-list
shares) and updates profiles/ncu_traffic.json (DRAM bytes per launch per kernel kind, read by
bench.py for the roofline "traffic" field).
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = {"0": "gemm_stats", "1": "gemm_grad", "2": "gemm_dw", "3": "gemm_dx", "4": "gemm_debug"}
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (sm__pipe)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor smem-read active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
]


def kind_of(name: str) -> str:
    if "lce_gemm_kernel<" in name:
        return KIND.get(name.split("<")[1].split(",")[0].strip(), "gemm?")
    if "lce_group_kernel<" in name:
        # <CG, NB>: NB = 4 staging buffers only for launches with a dW read-modify-write (the
        # schedule-S dW+dX group); NB = 2 for the stash / statistics GEMMs (slf_lce.cu launch_group)
        args = [x.strip() for x in name.split("<")[1].split(">")[0].split(",")]
        if len(args) >= 2:
            return "gemm_group" if args[1] == "4" else "gemm_stats"
        return "gemm (group kernel)"
    return name.split("(")[0].replace("void ", "").strip()


def to_bytes(v: str, unit: str) -> float:
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--note", default="")
    ap.add_argument("--rep-kinds", default="", help="comma list naming the captured GEMM launches in order")
    ap.add_argument("--split-ms", type=float, default=0.0,
                    help="label lce_group_kernel launches >= this many ms as gemm_group, shorter as gemm_stats")
    ap.add_argument("--launch-cycle", default="",
                    help="comma list naming consecutive lce_group_kernel launches of the launch list cyclically")
    a = ap.parse_args()
    rep_kinds = [k for k in a.rep_kinds.split(",") if k]
    cycle = [k for k in a.launch_cycle.split(",") if k]
    out = [f"# ncu summary {a.tag} ({a.config})", "", a.note, ""]
    traffic = {}
    if a.rep:
        raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        hdr, units, data = rows[0], rows[1], rows[2:]
        idx = {h: i for i, h in enumerate(hdr)}
        out += ["## `ncu --set full` capture (one launch per kernel kind; serialised, cold-ish cache)", "",
                "| kernel | " + " | ".join(k[1] for k in KEYS) + " |", "|---" * (len(KEYS) + 1) + "|"]
        for di, d in enumerate(data):
            k = rep_kinds[di] if di < len(rep_kinds) else kind_of(d[idx["Kernel Name"]])
            cells = []
            for m, _ in KEYS:
                if m in idx:
                    cells.append(f"{d[idx[m]]} {units[idx[m]]}".strip())
                else:
                    cells.append("n/a")
            out.append(f"| {k} | " + " | ".join(cells) + " |")
            if "dram__bytes_read.sum" in idx:
                tb = to_bytes(d[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]]) + \
                    to_bytes(d[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
                traffic.setdefault(k, tb)
        out.append("")
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 5]
        hdr = rows[0]
        agg = collections.defaultdict(lambda: [0, 0.0])
        gi = 0
        for r in rows[1:]:
            if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            k = kind_of(r[hdr.index("Kernel Name")])
            if cycle and "lce_group_kernel" in r[hdr.index("Kernel Name")]:
                k = cycle[gi % len(cycle)]
                gi += 1
            if a.split_ms and "lce_group_kernel" in r[hdr.index("Kernel Name")]:
                ms = float(r[hdr.index("Metric Value")].replace(",", "")) / 1e6
                k = "gemm_group" if ms >= a.split_ms else "gemm_stats"
            agg[k][0] += 1
            agg[k][1] += float(r[hdr.index("Metric Value")].replace(",", "")) / 1e6
        tot = sum(v[1] for v in agg.values())
        out += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, one step)", "",
                f"Total device time of the captured launches: {tot:.3f} ms (serialised, so compare shares).", "",
                "| kernel | launches | ms | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            out.append(f"| {k} | {v[0]} | {v[1]:.3f} | {v[1] / tot:.3f} |")
        out.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}.md"), "w") as f:
        f.write("\n".join(out))
    if traffic:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        cur = json.load(open(p)) if os.path.exists(p) else {}
        cur[a.config] = {**cur.get(a.config, {}), **traffic, "_source": f"profiles/ncu_{a.tag}.md"}
        json.dump(cur, open(p, "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()
