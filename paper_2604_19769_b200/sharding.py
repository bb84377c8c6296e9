"""Work partitioning across GPUs.

Streams are independent in the reference (one Engine per KV stream,
SPEC.md:113), so the decode path shards without any exchange inside
attention:

* head sharding (configs[3]): rank r of N owns KV heads [r*H/N, (r+1)*H/N) of
  every layer; its slow-tier records live in its own pinned arena and cross
  its own PCIe link.  The per-head outputs are all-gathered (NCCL over
  NVLink) because the next layer's o_proj needs every head.
* request sharding (configs[2] at N>1): rank r owns requests
  [r*R/N, (r+1)*R/N); no collective at all.

Global stream order is (request, layer, kv_head) row-major, matching the
S = layers x kv_heads x requests streams of one handle.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    layers: int
    kv_heads: int
    requests: int
    mode: str  # "heads" | "requests"

    def local_streams(self) -> List[int]:
        """Global stream ids owned by this rank, in local handle order."""
        L, H, R, N, r = self.layers, self.kv_heads, self.requests, self.world, self.rank
        if self.mode == "heads":
            if H % N:
                raise ValueError(f"{N} ranks do not divide {H} KV heads")
            h0, h1 = r * H // N, (r + 1) * H // N
            return [(q * L + l) * H + h for q in range(R) for l in range(L) for h in range(h0, h1)]
        if R % N:
            raise ValueError(f"{N} ranks do not divide {R} requests")
        q0, q1 = r * R // N, (r + 1) * R // N
        return [(q * L + l) * H + h for q in range(q0, q1) for l in range(L) for h in range(H)]

    @property
    def n_local(self) -> int:
        return self.layers * self.kv_heads * self.requests // self.world

    @property
    def needs_gather(self) -> bool:
        return self.mode == "heads" and self.world > 1


def gather_outputs(local_out, plan: ShardPlan, group=None):
    """All-gather per-head outputs [n_local, G, d] into global stream order
    [S, G, d] on every rank (head sharding).  Works on any torch.distributed
    backend (NCCL on the GPU box, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    N = plan.world
    if N == 1:
        return local_out
    src = local_out.contiguous()
    if src.is_cuda and dist.get_backend(group) != "nccl":
        src = src.cpu()  # gloo: stage through the host (test-only path)
    gathered = torch.empty((N * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype,
                           device=src.device)
    dist.all_gather_into_tensor(gathered, src, group=group)
    gathered = gathered.to(local_out.device)
    L, H, R = plan.layers, plan.kv_heads, plan.requests
    G, d = local_out.shape[1], local_out.shape[2]
    if plan.mode == "heads":
        # [N][R][L][H/N][G][d] -> [R][L][N][H/N][G][d]: rank-major -> head-major
        x = gathered.view(N, R, L, H // N, G, d).permute(1, 2, 0, 3, 4, 5)
    else:
        x = gathered.view(N, R // N, L, H, G, d)
    return x.reshape(R * L * H, G, d)


class PeerUnavailable(RuntimeError):
    """Some pair of ranks cannot map each other's memory (no P2P path)."""


def probe_peers(device: int, group=None) -> dict:
    """Exchange every rank's PCI bus id and check, on every rank, that its
    device can access every other rank's GPU (ttkv_peer_probe:
    cudaDeviceGetByPCIBusId + cudaDeviceCanAccessPeer).  Returns
    {"bus_ids": [...], "ok": bool, "failed": [(rank, peer), ...]}, identical on
    every rank."""
    import ctypes as C

    import torch.distributed as dist

    from . import _lib as L

    lib = L.lib()
    buf = C.create_string_buffer(32)
    from .engine import _check
    _check(lib.ttkv_pci_bus_id(device, buf, 32))
    me = buf.value.decode()
    world = dist.get_world_size(group)
    bus = [None] * world
    dist.all_gather_object(bus, me, group=group)
    rank = dist.get_rank(group)
    mine = []
    for r, b in enumerate(bus):
        ok = C.c_int(0)
        _check(lib.ttkv_peer_probe(device, b.encode(), C.byref(ok)))
        if not ok.value:
            mine.append((rank, r))
    failed = [None] * world
    dist.all_gather_object(failed, mine, group=group)
    failed = [p for f in failed for p in f]
    return {"bus_ids": bus, "ok": not failed, "failed": failed}


class PeerGather:
    """Combine fused with the all-gather over peer memory
    (ttkv_gpu_peer_gather_*, include/ttkv_gpu.h): every rank's combine kernel
    stores its (stream, head) rows straight into every rank's gathered buffer
    over NVLink (CUDA IPC mappings exchanged once through torch.distributed),
    so a decode step needs no separate collective.  Rows are in global stream
    order, like gather_outputs."""

    def __init__(self, engine, plan: ShardPlan, group=None):
        import ctypes as C

        import numpy as np
        import torch.distributed as dist

        from .engine import _check

        self.engine, self.plan = engine, plan
        # every pair must have a P2P path before any rank maps or publishes
        self.probe = probe_peers(engine.device, group)
        if not self.probe["ok"]:
            raise PeerUnavailable(f"no peer access between ranks {self.probe['failed']} "
                                  f"(bus ids {self.probe['bus_ids']})")
        self.S = plan.layers * plan.kv_heads * plan.requests
        self.shape = (self.S, engine.G, engine.config.d_v)
        lib = engine._lib
        gidx = np.ascontiguousarray(plan.local_streams(), np.uint32)
        if gidx.size != engine.S:
            raise ValueError("peer gather: the engine's streams do not match the shard plan")
        handle = (C.c_uint8 * 64)()
        _check(lib.ttkv_gpu_peer_gather_init(engine.handle, plan.world, plan.rank, self.S,
                                             gidx.ctypes.data_as(C.c_void_p), handle),
               engine.handle)
        handles = [None] * plan.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        blob = b"".join(handles)
        rc = lib.ttkv_gpu_peer_gather_open(engine.handle, blob)
        # every rank must map every peer, or none may publish (a rank on the
        # NCCL fallback would leave the others waiting for its rows)
        oks = [None] * plan.world
        dist.all_gather_object(oks, rc == 0, group=group)
        if not all(oks):
            lib.ttkv_gpu_peer_gather_close(engine.handle)
            _check(rc, engine.handle)
            raise RuntimeError("peer gather: a peer could not map the IPC buffers")
        self._C, self._np = C, np

    def device_ptr(self) -> int:
        C = self._C
        p = C.c_void_p()
        from .engine import _check
        _check(self.engine._lib.ttkv_gpu_peer_gather_output(self.engine.handle, C.byref(p), None),
               self.engine.handle)
        return p.value

    def host(self):
        """The last step's gathered rows [S][G][d_v] (float64) on the host;
        raises if a rank failed to arrive."""
        C, np = self._C, self._np
        from .engine import Error, _check
        p, t = C.c_void_p(), C.c_int()
        lib = self.engine._lib
        _check(lib.ttkv_gpu_peer_gather_output(self.engine.handle, C.byref(p), C.byref(t)),
               self.engine.handle)
        if t.value:
            raise Error("peer gather: a rank did not deliver its rows")
        return self._view(p.value).cpu().numpy()

    def verify(self, local_out, group=None) -> tuple:
        """Self-check after a decode step, on every rank together: the rows
        the combine kernels stored over peer memory equal an NCCL (or gloo)
        all-gather of this rank's own output (`local_out`, [S_local][G][d_v]).
        Returns (ok, reason), identical on every rank."""
        import torch.distributed as dist
        try:
            peer = self.host()
            ref = gather_outputs(local_out, self.plan, group).cpu().numpy()
            mine = (bool(self._np.array_equal(peer, ref)), "" if self._np.array_equal(peer, ref)
                    else "gathered rows differ from the collective's")
        except Exception as e:  # noqa: BLE001 -- a rank that timed out or failed
            mine = (False, repr(e))
        res = [None] * self.plan.world
        dist.all_gather_object(res, mine, group=group)
        bad = [f"rank {r}: {why}" for r, (ok, why) in enumerate(res) if not ok]
        return (not bad, "; ".join(bad))

    def close(self):
        """Stop storing rows into the peers (the combine writes locally only)."""
        from .engine import _check
        _check(self.engine._lib.ttkv_gpu_peer_gather_close(self.engine.handle), self.engine.handle)

    def tensor(self):
        """Zero-copy torch view of the last step's gathered rows on the device."""
        return self._view(self.device_ptr())

    def _view(self, ptr):
        import torch

        class _Rows:
            pass

        rows = _Rows()
        rows.__cuda_array_interface__ = {"shape": self.shape, "typestr": "<f8",
                                         "data": (ptr, False), "version": 3, "strides": None}
        return torch.as_tensor(rows, device=torch.device("cuda", self.engine.device))
