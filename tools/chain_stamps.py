"""Where one layer of layer-sequential decode spends its time, from %globaltimer
stamps inside the kernels (the measurement-only library of `make stamps`,
build/stamps/libttkv_gpu.so; not the bench contract).

  python tools/chain_stamps.py [layers] [tokens]

Per layer (one handle: 8 streams x 4 heads, 128K, slow tier in HBM), relative
to the previous layer's combine end, the medians of:
  selection: entry, centroids staged, after its programmatic wait + q,
  scored, cluster barrier, keys gathered, radix, second barrier, union;
  record kernel: entry, after its programmatic wait (= selection complete);
  combine: entry, after its wait (= record kernel complete), end (last CTA).
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_19769_b200._lib as L  # noqa: E402

L.LIB_PATH = os.path.join(ROOT, "build", "stamps", "libttkv_gpu.so")
import torch  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def read(lib, name, n):
    buf = np.zeros((n, 16), np.uint64)
    cnt = C.c_uint()
    fn = getattr(lib, f"ttkv_dbg_read_{name}")
    fn.argtypes = [C.c_void_p, C.c_uint, C.POINTER(C.c_uint)]
    assert fn(buf.ctypes.data, n, C.byref(cnt)) == 0
    return buf, cnt.value


def main():
    Lyr = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    tokens = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    S = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    G = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    ctx = int(sys.argv[5]) if len(sys.argv) > 5 else 131072
    D = 128
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=128)
    engs = []
    for layer in range(Lyr):
        e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, 0.45), n_streams=S, heads_per_stream=G,
                                device=0, reserve_tokens=ctx + 512, slow_tier=1)
        e.set_stream(stream.cuda_stream)
        e.prefill_synthetic(ctx, seed=7000 + layer)
        engs.append(e)
    lib = L.lib()
    assert "stamps" in lib._name, lib._name
    qs = [torch.randn(S, G, D, device=dev) for _ in range(Lyr)]
    ks = [torch.randn(S, D, device=dev).half() for _ in range(Lyr)]
    vs = [torch.randn(S, D, device=dev).half() for _ in range(Lyr)]
    outs = [torch.empty(S, G, D, device=dev, dtype=torch.float64) for _ in range(Lyr)]

    def token():
        for layer, e in enumerate(engs):
            e.decode_step_device(qs[layer].data_ptr(), ks[layer].data_ptr(), vs[layer].data_ptr(),
                                 outs[layer].data_ptr(), dtype=1)
    torch.cuda.synchronize()
    _, s0 = read(lib, "sel", 1)
    _, w0 = read(lib, "slow", 1)
    _, c0 = read(lib, "comb", 1)
    _, f0 = read(lib, "fast", 1)
    torch.cuda._sleep(int(1.9e9 * 0.05))  # the host runs ahead: a device-bound chain
    for _ in range(tokens):
        token()
    torch.cuda.synchronize()
    sel, s1 = read(lib, "sel", 4096)
    slow, w1 = read(lib, "slow", 4096)
    comb, c1 = read(lib, "comb", 4096)
    fast, f1 = read(lib, "fast", 4096)
    n = s1 - s0
    assert n == w1 - w0 == c1 - c0 == Lyr * tokens, (s1 - s0, w1 - w0, c1 - c0)
    rows = []
    for i in range(1, n):  # layer i relative to layer i-1's combine end
        t0 = float(comb[(c0 + i - 1) % 4096, 15])
        si, wi, ci = (s0 + i) % 4096, (w0 + i) % 4096, (c0 + i) % 4096
        fi = (f0 + i) % 4096
        rows.append([sel[si, k] - t0 for k in range(8)] +
                    [slow[wi, 0] - t0, slow[wi, 1] - t0,
                     comb[ci, 0] - t0, comb[ci, 1] - t0, comb[ci, 15] - t0,
                     fast[fi, 0] - t0, (fast[fi, 15] - t0) if fast[fi, 15] else np.nan])
    r = np.nanmedian(np.array(rows, dtype=np.float64), axis=0) / 1e3
    names = ["sel entry", "sel staged+wait+q", "sel scored", "sel barrier 1", "sel gathered",
             "sel radix", "sel barrier 2", "sel union done", "slow entry", "slow after wait",
             "comb entry", "comb after wait", "comb end", "fast entry",
             "fast done (device join)"]
    cta = np.zeros((1024, 8), np.uint64)
    fn = lib.ttkv_dbg_read_slow_cta
    fn.argtypes = [C.c_void_p]
    assert fn(cta.ctypes.data) == 0
    grid = int(np.count_nonzero(cta[:, 1]))
    cta = cta[:grid].astype(np.float64)
    t0 = cta[:, 1].min()
    print(f"# record kernel, the last launch: {grid} CTAs, records per CTA "
          f"min {cta[:, 5].min():.0f} median {np.median(cta[:, 5]):.0f} max {cta[:, 5].max():.0f}; "
          "us after the first CTA's wait returns (median / max over CTAs)")
    busy = cta[:, 5] > 0  # CTAs with records (the rest stamp no record phases)
    for k, nm in [(0, "entry"), (1, "after wait"), (2, "schedule done"), (3, "first record in smem"),
                  (4, "last partial written")]:
        v = (cta[busy if k >= 3 else slice(None), k] - t0) / 1e3
        print(f"  {nm:22s} {np.median(v):8.2f} {v.max():8.2f}  (min {v.min():.2f})")
    per = (cta[busy, 4] - cta[busy, 3]) / 1e3 / np.maximum(cta[busy, 5] - 1, 1)
    print(f"  us per record after the first: median {np.median(per):.2f}")
    print(f"# layer-sequential chain, {Lyr} layers x {tokens} tokens, medians over {n - 1} layers,")
    print("# us after the previous layer's combine end (%globaltimer, measurement build)")
    for nm, v in zip(names, r):
        print(f"  {nm:22s} {v:8.2f}")


if __name__ == "__main__":
    main()
