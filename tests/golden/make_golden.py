"""Generate the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref/libttkv_ref.so, built from /root/reference by oracle/Makefile).

  criterion3.json   acceptance.cpp:172-195 operating point: per-step fetched
                    lists, fp64 outputs and the H->G total (seed 3, 16K ctx).
  blocks_small.json serialize_block bytes (quantizer.cpp:248-274) of every
                    slow block after a seeded prefill.
  needle.json       criterion 7 (acceptance.cpp:376-426) hit/miss per seed for
                    the first 100 seeds at B=128 and B=256.
Run: python tests/golden/make_golden.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _oracle as O  # noqa: E402


def criterion3():
    pk, pv, dk, dv, dq = O.generate_workload(16384, 8, 128, 128, 3, use_ref=True)
    r = O.RefEngine(1024 * 256 * 2, 128, 128, 128)
    r.prefill(pk, pv)
    out = {"fetched": [], "outputs": [], "total_h2g_bytes": 0.0}
    for t in range(8):
        x = r.decode_step(dq[t], dk[t], dv[t])
        out["fetched"].append([int(i) for i in x["fetched"]])
        out["outputs"].append([float(v) for v in x["output"]])
        out["total_h2g_bytes"] += x["bytes_transferred"]
    tot = C.c_uint64()
    out["harness_traffic_reduction"] = O.ref().ref_traffic_reduction(C.byref(tot))
    out["harness_total_h2g_bytes"] = tot.value
    return out


def blocks_small():
    g = dict(ctx=700, d=16, B=32, l_fast=128, kb=8, vb=4, seed=21)
    pk, pv, *_ = O.generate_workload(g["ctx"], 1, g["d"], g["d"], g["seed"], use_ref=True)
    r = O.RefEngine(g["l_fast"] * 2 * g["d"] * 2, g["d"], g["d"], g["B"], g["kb"], g["vb"])
    r.prefill(pk, pv)
    g["blocks_hex"] = [r.serialize_block(i).hex() for i in range(r.slow_blocks())]
    return g


def needle():
    out = {}
    q = np.full(64, 1 / 8, np.float32)
    for B in (128, 256):
        hits = []
        for t in range(100):
            pk, pv, *_ = O.generate_workload(4096, 0, 64, 1, 40000 + t, needle=True, use_ref=True)
            r = O.RefEngine(1024 * 65 * 2, 64, 1, B)
            r.prefill(pk, pv)
            n = r.slow_blocks()
            # score/select through the reference API on the reference's centroids
            # (decoded from its serialized blocks)
            scores = []
            for i in range(n):
                blob = r.serialize_block(i)
                off = 4 + 2 + 24 + 12 + 4 + 8 * (64 + 1)
                cen = np.frombuffer(blob[off:off + 256], np.float32)
                scores.append(O.ref().ref_score_block(q, np.ascontiguousarray(cen), 64))
            ids = np.arange(n, dtype=np.uint64)
            sel = np.zeros(n, np.uint64)
            k = O.ref().ref_select_top_k(np.array(scores), ids, n, 0, 0, 0.45, sel)
            hits.append(int((256 // B) in sel[:k]))
        out[str(B)] = hits
    return out


if __name__ == "__main__":
    for name, fn in [("criterion3.json", criterion3), ("blocks_small.json", blocks_small),
                     ("needle.json", needle)]:
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(fn(), f)
        print("wrote", name)
