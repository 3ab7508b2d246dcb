#!/usr/bin/env python
"""Pipeline trace of the GEMM kernels (aqb_gemm_trace): per-CTA clock64 stamps of the last of 8
back-to-back launches in a CUDA graph (the `scripts/gemm_bench.py` harness), summarised as
cycles from the PDL wait: first k-block consumed, median k-block interval, tile epilogue
start/end, drain; plus the entry/exit spread of the CTAs (globaltimer, ns).

    AQB_BUILD_DEFINES=-DAQB_GEMM_TRACE python -c "from paper_2505_10584_b200 import build; build.build(force=True)"
    python scripts/gemm_trace.py proj 1950 2048 2048 [more cases as name m n k ...]

(the stamps are compiled in only by that build; rebuild without the define afterwards)
"""

import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10584_b200 import _native, ops  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gemm_bench  # noqa: E402


def trace_case(name, m, n, k):
    tr = torch.zeros(4096 * 128, dtype=torch.int64, device="cuda")
    _native.call("aqb_gemm_trace", tr.data_ptr())  # raises unless a trace build
    try:
        r = gemm_bench.case(name, m, n, k)
    finally:
        _native.call("aqb_gemm_trace", None)
    torch.cuda.synchronize()
    t = tr.view(-1, 128).cpu()
    ctas = [i for i in range(t.shape[0]) if int(t[i, 0]) != 0]
    rows = []
    for c in ctas:
        s = [int(x) for x in t[c]]
        w = s[3]
        ks = [s[8 + i] for i in range(96) if s[8 + i] != 0]
        d = [b - a for a, b in zip(ks, ks[1:])]
        ep = [(s[104 + 2 * j] - w, s[105 + 2 * j] - w) for j in range(8) if s[104 + 2 * j] != 0]
        rows.append({"cta": c, "setup": s[2] - s[0], "pdl_wait": w - s[2],
                     "pro": [s[i] - s[0] if s[i] else None for i in (4, 6, 7)],  # init, alloc, cluster sync
                     "first_k": (ks[0] - w) if ks else None, "last_k": (ks[-1] - w) if ks else None,
                     "k_blocks": len(ks), "k_med": statistics.median(d) if d else None,
                     "k_max": max(d) if d else None, "epi": ep, "drained": s[120] - w if s[120] else None,
                     "g_entry": s[1], "g_exit": s[121]})
    ge = [x["g_entry"] for x in rows if x["g_entry"]]
    gx = [x["g_exit"] for x in rows if x["g_exit"]]
    mma = [x for x in rows if x["k_blocks"] > 0]

    def med(key):
        v = [x[key] for x in mma if x[key] is not None]
        return statistics.median(v) if v else None

    out = {"name": name, "m": m, "n": n, "k": k, "us_in_graph": r["us"], "ctas": len(rows),
           "mma_ctas": len(mma), "median": {key: med(key) for key in
                                            ("setup", "pdl_wait", "first_k", "last_k", "k_blocks", "k_med",
                                             "k_max", "drained")},
           "entry_spread_ns": (max(ge) - min(ge)) if ge else None,
           "exit_spread_ns": (max(gx) - min(gx)) if gx else None,
           "span_ns": (max(gx) - min(ge)) if ge and gx else None,
           "cta0": mma[0] if mma else None}
    print(json.dumps(out), flush=True)


def main():
    a = sys.argv[1:]
    for i in range(0, len(a), 4):
        trace_case(a[i], int(a[i + 1]), int(a[i + 2]), int(a[i + 3]))


if __name__ == "__main__":
    main()
