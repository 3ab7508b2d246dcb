#!/usr/bin/env python
"""Summarise ncu artefacts into small text files for profiles/.

    python scripts/ncu_summary.py report <file.ncu-rep>   # per-kernel key metrics (--set full capture)
    python scripts/ncu_summary.py launches <file.csv>     # launch-list time shares (gpu__time_duration pass)
    python scripts/ncu_summary.py sass <file.ncu-rep>     # executed-instruction mix + top stall sites
"""

import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu(mufu)_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_%"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct", "stall_long_sb_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_pipe_%"),
]


def _name(n):
    return re.sub(r"\(CUtensorMap.*", "", n.replace("void ", "").replace("aqb::", ""))


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    print(f"# ncu --set full summary: {path}")
    for r in rows[2:]:
        print(f"\n## {_name(r[h.index('Kernel Name')])}")
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                print(f"  {label:22s} {r[i]} {u[i]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        k = re.sub(r"<.*|\(.*", "", r[ik]).replace("void ", "").replace("aqb::", "")
        tot[k] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        cnt[k] += 1
    T = sum(tot.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none): {path}")
    print(f"# {sum(cnt.values())} launches, {T / 1e6:.3f} ms total (cold-cache, serialised: compare shares)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:40s} {cnt[k]:6d} {v / 1e6:10.3f} ms {100 * v / T:6.1f}%")




def sass(path, top=20):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    data = [r for r in rows[2:] if len(r) >= len(h)]
    ex, st = collections.Counter(), collections.Counter()
    for r in data:
        src = r[ix["Source"]].strip().split()
        op = (src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")).split(".")[0]
        ex[op] += int(r[ix["Instructions Executed"]] or 0)
        st[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot, tots = sum(ex.values()), sum(st.values())
    print(f"# executed warp instructions: {tot}; stall samples: {tots}")
    print("## instruction mix (executed share, stall-sample share)")
    for op, c in ex.most_common(top):
        print(f"  {op:10s} {c / tot * 100:5.1f}%  {st[op] / max(tots, 1) * 100:5.1f}%")
    print("## top stall sites")
    a0 = int(data[0][0], 16)
    for r in sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        print(f"  +{int(r[0], 16) - a0:#07x} {n / max(tots, 1) * 100:5.1f}%  exec {r[ix['Instructions Executed']]:>12s}  "
              f"{r[ix['Source']].strip()[:60]}")


if __name__ == "__main__":
    {"report": report, "launches": launches, "sass": sass}[sys.argv[1]](sys.argv[2])
