"""Static SASS of the product library's kernels (cuobjdump, no GPU needed).

  python tools/kernel_sig.py hist [lib.so] [kernel-substring ...]   opcode histograms
  python tools/kernel_sig.py sig  [lib.so] [kernel-substring ...]   SASS signatures

`sass_by_kernel` splits `cuobjdump -sass` into one text per kernel (mangled
name); `kernel_sig` hashes a kernel's SASS, so a measurement taken on one
build (profiles/traffic.json) can be checked against the kernel that is loaded
now -- it stays valid across rebuilds that do not change that kernel's code.
"""
import hashlib
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_19769_b200", "lib", "libttkv_gpu.so")
_INSN = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_.]*)")


def _cuobjdump():
    for c in ("cuobjdump", "/usr/local/cuda/bin/cuobjdump"):
        try:
            subprocess.run([c, "--version"], capture_output=True, check=True)
            return c
        except (OSError, subprocess.CalledProcessError):
            continue
    raise RuntimeError("cuobjdump not found")


def sass_by_kernel(lib=LIB):
    out = subprocess.run([_cuobjdump(), "-sass", lib], capture_output=True, text=True,
                         check=True).stdout
    kernels, name, buf = {}, None, []
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if name:
                kernels[name] = "\n".join(buf)
            name, buf = m.group(1), []
        elif name:
            buf.append(line)
    if name:
        kernels[name] = "\n".join(buf)
    return kernels


def _select(kernels, sub):
    """Kernels named `sub` (every template instantiation; a full mangled
    name selects exactly that one)."""
    if sub.startswith("_Z"):
        return {k: v for k, v in kernels.items() if k == sub}
    pat = re.compile(r"\d" + re.escape(sub) + r"[IE]")
    return {k: v for k, v in kernels.items() if pat.search(k)}


def kernel_sig(sub, lib=LIB):
    """sha256[:16] of the SASS of every kernel matching `sub` (sorted by name)."""
    ks = _select(sass_by_kernel(lib), sub)
    if not ks:
        return None
    h = hashlib.sha256()
    for k in sorted(ks):
        h.update(k.encode())
        h.update(ks[k].encode())
    return h.hexdigest()[:16]


def opcodes(text):
    c = Counter()
    for line in text.splitlines():
        m = _INSN.search(line)
        if m:
            c[m.group(2)] += 1
    return c


# bulk/tensor async copies, mbarrier ops, tensor-core MMAs, TMEM, PDL
KEY_OPS = {"UBLKCP", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKPF", "SYNCS", "HMMA", "IMMA", "UTCHMMA",
           "UTCMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "LDSM", "ACQBULK", "CREDUX", "REDUX",
           "LDGSTS", "LDGDEPBAR", "UCGABAR_ARV", "UCGABAR_WAIT", "ELECT", "FENCE", "CCTL",
           "MEMBAR", "ERRBAR"}


def hist(sub, lib=LIB, top=40):
    lines = []
    for name, text in sorted(_select(sass_by_kernel(lib), sub).items()):
        c = opcodes(text)
        base = Counter()
        for op, n in c.items():
            base[op.split(".")[0]] += n
        tot = sum(c.values())
        lines.append(f"== {name}  ({tot} SASS instructions, static)")
        key = {op: n for op, n in c.items() if op.split(".")[0] in KEY_OPS}
        lines.append("  Blackwell / async-copy / tensor ops: " +
                     (", ".join(f"{o} {n}" for o, n in sorted(key.items())) or "none"))
        lines.append("  by base opcode: " + ", ".join(f"{o} {n}" for o, n in base.most_common(top)))
        lines.append("  full opcodes:")
        for op, n in c.most_common(top):
            lines.append(f"    {op:34s} {n}")
    return "\n".join(lines)


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "hist"
    lib = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2].endswith(".so") else LIB
    subs = [a for a in sys.argv[2:] if not a.endswith(".so")] or ["slow_attn_kernel"]
    for s in subs:
        print(hist(s, lib) if mode == "hist" else f"{s} {kernel_sig(s, lib)}")
