"""Calibrate the reference's timing model (sim.cpp simulate_pipelined /
simulate_serial, restated in harness.py) with measured B200 rates and compare
its predictions with measured decode steps.

For each workload, with the slow tier in pinned host DRAM:
  1. the serial schedule (bulk gather of all selected records over PCIe into
     HBM, then attention) gives the two lane rates independently:
     transfer s/record = gather kernel time / records, compute s/record =
     slow-attention kernel time / records, fast-tier compute = fast kernel time;
  2. the model predicts the pipelined and the serial step from those rates
     (plus the measured append/score/select/combine prologue, which the
     reference's model does not contain);
  3. the pipelined engine (the product schedule) is measured and compared.
  python tools/calibrate_sim.py [steps] > profiles/r1_sim_calibration.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402
from paper_2604_19769_b200 import harness as H  # noqa: E402

WORK = {
    "cfg1": dict(S=32, G=1, ctx=32768),
    "cfg2": dict(S=256, G=4, ctx=131072),
    "cfg3": dict(S=4096, G=4, ctx=32768),
}


def run(S, G, ctx, serial, steps):
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 256 * 2, d_k=128, d_v=128, block_size=128)
    eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=ctx + 512,
                              serial_schedule=serial)
    eng.prefill_synthetic(ctx, seed=5)
    rng = np.random.default_rng(0)
    q = rng.standard_normal((S, G, 128)).astype(np.float32)
    kn = rng.standard_normal((S, 128)).astype(np.float16)
    vn = rng.standard_normal((S, 128)).astype(np.float16)
    eng.decode_step(q, kn, vn)  # warm-up
    eng.set_timing(True)
    eng.kernel_times(reset=True)
    for _ in range(steps):
        r = eng.decode_step(q, kn, vn)
    kt = eng.kernel_times(reset=True)
    eng.close()
    per = {k[3:]: v / steps for k, v in kt.items() if k.startswith("ms_")}
    return per, r.union_blocks


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    for name, w in WORK.items():
        ser, union = run(w["S"], w["G"], w["ctx"], True, steps)
        pipe, union_p = run(w["S"], w["G"], w["ctx"], False, steps)
        t_rec = ser["gather"] / union * 1e-3
        c_rec = ser["slow"] / union * 1e-3
        model = H.calibrated_step(ser["fast"] * 1e-3, union, c_rec, t_rec)
        prologue = pipe["append"] + pipe["score"] + pipe["select"] + pipe["combine"]
        pred_pipe = model["pipelined_ms"] + prologue
        pred_ser = model["serial_ms"] + ser["append"] + ser["score"] + ser["select"] + \
            ser["combine"]
        print(json.dumps({
            "workload": name, **w, "records_per_step": union,
            "measured_rates": {"transfer_gbs": union * 24576 / (ser["gather"] * 1e-3) / 1e9,
                               "compute_records_per_s": union / (ser["slow"] * 1e-3),
                               "fast_ms": ser["fast"]},
            "model": model,
            "pipelined": {"predicted_ms": pred_pipe, "measured_ms": pipe["step"],
                          "ratio": pipe["step"] / pred_pipe},
            "serial": {"predicted_ms": pred_ser, "measured_ms": ser["step"],
                       "ratio": ser["step"] / pred_ser,
                       # the B200 serial schedule runs the fast tier on its own
                       # stream next to the slow attention (both after the
                       # gather); the model's compute lane serializes them
                       "predicted_fast_concurrent_ms":
                           pred_ser - min(ser["fast"], ser["slow"])},
            "measured_pipelining_gain": ser["step"] / pipe["step"],
            "kernels_ms": {"serial": ser, "pipelined": pipe},
        }), flush=True)


if __name__ == "__main__":
    main()
