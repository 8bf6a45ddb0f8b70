"""Summarise ncu captures into profiles/ (tracked): launch-list shares and the
full-capture metrics of the top kernels.

    python tools/profile_summary.py --launches gpurun_out/launches.csv \
        --full gpurun_out/prof_full.ncu-rep --tag r1 [--bench gpurun_out/bench.json]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
NCU = "/usr/local/cuda/bin/ncu"

METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    # DMMA (mma.sync f64) issues to the tensor pipe, not the fp64 pipe counter above
    "dmma_pipe_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "registers_per_thread": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block_static",
    "grid_size": "launch__grid_size",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "red_sectors_to_l2": "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
}
STALLS = "smsp__average_warps_issue_stalled_"


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    tot = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > mi:
            tot[r[ki]].append(float(r[mi].replace(",", "")))
    total = sum(sum(v) for v in tot.values())
    out = []
    for k, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k[:100], "launches": len(v), "total_us": sum(v) / 1e3, "mean_us": sum(v) / len(v) / 1e3,
                    "share": sum(v) / total})
    return out


def full_metrics(rep):
    raw = subprocess.run([NCU, "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        m = {"kernel": d["Kernel Name"][:100]}
        for k, name in METRICS.items():
            try:
                m[k] = float(d.get(name, "nan").replace(",", ""))
            except ValueError:
                m[k] = None
        st = {}
        for k in h:
            if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio"):
                try:
                    st[k[len(STALLS):-len("_per_issue_active.ratio")]] = float(d[k])
                except ValueError:
                    pass
        m["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1])[:6])
        res.append(m)
    units = dict(zip(h, rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "ms": 1e-3, "msecond": 1e-3, "s": 1.0}
    for m in res:
        rb = m.get("dram_read_bytes") or 0.0
        wb = m.get("dram_write_bytes") or 0.0
        m["dram_bytes_per_launch"] = (rb * scale.get(units.get(METRICS["dram_read_bytes"], "byte"), 1.0)
                                      + wb * scale.get(units.get(METRICS["dram_write_bytes"], "byte"), 1.0))
        d = m.get("duration_ns")
        if d is not None:
            m["duration_s"] = d * scale.get(units.get(METRICS["duration_ns"], "ns"), 1e-9)
    return res, {k: units.get(v, "") for k, v in METRICS.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--bench")
    ap.add_argument("--tag", default="r1")
    a = ap.parse_args()
    outdir = ROOT / "profiles"
    outdir.mkdir(exist_ok=True)
    data = {}
    md = [f"# Profile summary {a.tag}\n"]
    if a.bench:
        b = json.loads(Path(a.bench).read_text().strip().splitlines()[-1])
        data["bench"] = b
        md.append(f"bench: {b['value']:.1f} {b['unit']} ({b['ms_per_step']:.3f} ms/step), e2e "
                  f"{b.get('e2e', {}).get('value', float('nan')):.1f}, roofline frac "
                  f"{b.get('roofline', {}).get('frac', float('nan')):.3f} ({b.get('roofline', {}).get('kernel')}), "
                  f"clocks {b.get('clocks')}\n")
    if a.launches:
        ls = launch_shares(a.launches)
        data["launch_list"] = ls
        md.append("## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n")
        md.append("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
        for x in ls[:15]:
            md.append(f"| `{x['kernel'][:70]}` | {x['launches']} | {x['total_us']:.1f} | {x['mean_us']:.1f} | {x['share']:.1%} |")
        md.append("")
    if a.full:
        fm, units = full_metrics(a.full)
        data["full"] = fm
        data["full_units"] = units
        md.append("## Full capture (ncu --set full), per launch\n")
        for m in fm:
            md.append(f"### `{m['kernel']}`\n")
            for k in METRICS:
                md.append(f"- {k}: {m[k]} {units.get(k, '')}")
            md.append(f"- dram bytes per launch (read + write): {m['dram_bytes_per_launch']:.4g}")
            md.append(f"- top stalls (per issued instruction): {m['stalls_per_issue']}\n")
    (outdir / f"{a.tag}_summary.json").write_text(json.dumps(data, indent=1))
    (outdir / f"{a.tag}_summary.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
