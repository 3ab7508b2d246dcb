"""Golden vectors for the geometry boundary (``Bucket``, ``LatentShape``, ``token_count``,
``snap_bucket``) and the planner leftovers (``resolved_param_count``, ``load_chunk_table``)
from the REAL reference (``ditplan``).

Run in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden_buckets.py

Records ``buckets.py:33-122`` over a grid of buckets x VAE specs x patch sizes (incl. the
DimensionError cases), ``config.py:252-256`` over supplied / estimated param counts, and
``memory.py:110-134`` over valid and malformed chunk-table documents.  The GPU box never
reads ``/root/reference``.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "buckets.json")

CHUNK_DOCS = [
    {"chunks": [{"name": "flash_attention", "coeff_bsh": 2, "coeff_bas": 64, "fwd_latency_ms": 127.5}],
     "ref_seqlen": 4096, "ref_tp": 4},
    {"chunks": [{"name": "a", "coeff_bsh": 1.5}, {"name": "b", "coeff_bsh": 2, "recomputable": False,
                                                  "offloadable": False}], "ref_batch": 2, "ref_hidden": 1024,
     "ref_heads": 8, "ignored_top_level": 1},
    {"chunks": []},
    {"chunks": [{"coeff_bsh": 1}]},
    {"chunks": [{"name": "a", "coeff_bsh": 1, "speed": 3}]},
    {"chunks": [{"name": "a", "coeff_bsh": 1, "zz": 1, "aa": 2}]},
    {"chunks": [{"name": "a", "coeff_bsh": -1}]},
    {"chunks": [{"name": "a", "coeff_bsh": 1, "fwd_latency_ms": 0}]},
    {"chunks": [{"name": "a", "coeff_bsh": 1}, {"name": "a", "coeff_bsh": 2}]},
    {"chunk": []},
    [1, 2, 3],
    "not json {",
]


def main():
    sys.path.insert(0, REF)
    from ditplan.buckets import Bucket, VaeSpec, snap_bucket, token_count
    from ditplan.config import ModelArch, resolved_param_count
    from ditplan.errors import ConfigError, DimensionError
    from ditplan.memory import load_chunk_table

    cases = []
    vaes = [VaeSpec(), VaeSpec(temporal_ratio=8, spatial_ratio=16, latent_channels=16), VaeSpec(1, 1, 4)]
    patches = [None, (1, 2, 2), (2, 2, 2), (1, 1, 1), (2, 4, 3)]
    videos = [(1, 8, 8), (17, 480, 832), (61, 480, 848), (61, 480, 854), (129, 720, 1280), (125, 720, 1280),
              (5, 64, 64), (9, 16, 48), (33, 256, 256), (18, 480, 832), (17, 481, 832), (17, 480, 833), (97, 544, 960)]
    for vi, vae in enumerate(vaes):
        for p in patches:
            arch = None if p is None else ModelArch(hidden_size=64, num_heads=4, num_layers=2, patch_t=p[0],
                                                    patch_h=p[1], patch_w=p[2])
            for batch in (1, 3):
                for f, h, w in videos:
                    b = Bucket(batch, f, h, w)
                    rec = {"vae": vi, "patch": p, "bucket": [batch, f, h, w], "label": b.label()}
                    try:
                        ls = token_count(b, vae, arch)
                        rec["shape"] = [ls.t_lat, ls.h_lat, ls.w_lat, ls.tokens, ls.tokens_batch]
                    except DimensionError as e:
                        rec["error"] = [str(e), e.path]
                    sb = snap_bucket(b, vae, arch)
                    rec["snapped"] = list(sb.key())
                    cases.append(rec)
    bucket_errors = []
    for kw in ({"batch": 0, "frames": 1, "height": 8, "width": 8}, {"batch": 1, "frames": 0, "height": 8, "width": 8},
               {"batch": 1, "frames": 1, "height": -8, "width": 8}, {"batch": 1, "frames": 1, "height": 8, "width": 0}):
        try:
            Bucket(**kw)
        except ConfigError as e:
            bucket_errors.append({"kwargs": kw, "error": str(e), "path": e.path})
    params = []
    for H, A, L, pc in ((2048, 16, 28, None), (3072, 24, 54, 13.4e9), (3072, 24, 54, None), (128, 4, 2, 1234.0)):
        for mode in ("shared-weights", "per-block-dedicated"):
            arch = ModelArch(hidden_size=H, num_heads=A, num_layers=L, adaln_mode=mode, param_count=pc)
            params.append({"dims": [H, A, L, mode, pc], "value": resolved_param_count(arch)})
    tables = []
    with tempfile.TemporaryDirectory() as d:
        for k, doc in enumerate(CHUNK_DOCS):
            path = os.path.join(d, f"t{k}.json")
            with open(path, "w") as fh:
                fh.write(doc if isinstance(doc, str) else json.dumps(doc))
            rec = {"doc": doc}
            try:
                t = load_chunk_table(path)
                rec["table"] = {"chunks": [c.__dict__ for c in t.chunks],
                                **{m: getattr(t, m) for m in ("ref_batch", "ref_seqlen", "ref_hidden", "ref_heads",
                                                              "ref_tp")}}
            except ConfigError as e:
                rec["error"] = {"str": str(e).replace(path, "<file>"), "path": e.path.replace(path, "<file>")}
            tables.append(rec)
        try:
            load_chunk_table(os.path.join(d, "missing.json"))
        except ConfigError as e:
            tables.append({"missing": True, "path_is_file": e.path == os.path.join(d, "missing.json"),
                           "starts": str(e).split(":")[0] == os.path.join(d, "missing.json")})
    with open(OUT, "w") as fh:
        json.dump({"token_count": cases, "bucket_errors": bucket_errors, "resolved_param_count": params,
                   "chunk_tables": tables}, fh, indent=0)
    print(f"wrote {OUT}: {len(cases)} token_count cases, {len(tables)} chunk-table docs")


if __name__ == "__main__":
    main()
