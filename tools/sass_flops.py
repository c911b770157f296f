"""Hardware FP32 flops per P2P pair, counted from the built library's SASS.

ncu's smsp__sass_thread_inst_executed_op_{fadd,fmul,ffma} counters do not count
the packed FP32x2 instructions (FADD2/FMUL2/FFMA2) the sm_100a kernels use, so
bench.py derives the per-pair hardware flop count statically instead: it finds
the two source loops of k_p2p (backward branches), counts FADD2 + FMUL2 +
2 FFMA2 per loop body (+ scalar FADD/FMUL/FFMA), excludes forward-branched
blocks inside the body (the close-pair series, only taken when some lane has
rho < 0.8), and divides by the pairs the body evaluates (two LDS.128 per
source, three for the near kernel; two targets per lane).  Returns {"near": F_near, "far": F_far}.
"""
from __future__ import annotations

import re
import subprocess


def _sass(lib, func_regex="k_p2p"):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    body, on = [], False
    for line in out.split("\n"):
        if "Function :" in line:
            on = re.search(func_regex, line) is not None
            continue
        if on:
            m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
            if m:
                body.append((int(m.group(1), 16), m.group(2).strip()))
    return body


def _op(ins):
    parts = ins.split()
    if parts[0].startswith("@"):
        parts = parts[1:]
    return parts[0], parts


def p2p_flops_per_pair(lib):
    ins = _sass(lib)
    loops = []
    for addr, text in ins:
        op, parts = _op(text)
        if op.startswith("BRA"):
            tgt = [p for p in parts if p.startswith("0x")]
            if tgt:
                t = int(tgt[-1].rstrip(","), 16)
                if t < addr:
                    loops.append((t, addr))
    # innermost loops only (a source loop contains no other loop)
    loops = [(lo, hi) for lo, hi in loops
             if not any((a, b) != (lo, hi) and lo <= a and b <= hi for a, b in loops)]
    res = {}
    for lo, hi in loops:
        body = [(a, t) for a, t in ins if lo <= a <= hi]
        ops = [_op(t)[0] for _, t in body]
        if not any(o.startswith("FFMA2") for o in ops) or not any(o.startswith("LDS.128") for o in ops):
            continue
        # forward-branched blocks inside the body
        skip = []
        for a, t in body:
            op, parts = _op(t)
            if op.startswith("BRA") and t.startswith("@"):
                tgt = [p for p in parts if p.startswith("0x")]
                if tgt:
                    x = int(tgt[-1].rstrip(","), 16)
                    if a < x <= hi:
                        skip.append((a, x))
        cnt = {}
        for a, t in body:
            if any(s < a < e for s, e in skip):
                continue
            o = _op(t)[0].split(".")[0]
            cnt[o] = cnt.get(o, 0) + 1
        kind = "near" if "MUFU" in "".join(t for _, t in body) and any("EX2" in t for _, t in body) else "far"
        sources = cnt.get("LDS", 0) // (3 if kind == "near" else 2)   # q, a (+ c for the near kernel)
        if sources == 0:
            continue
        packed = cnt.get("FADD2", 0) + cnt.get("FMUL2", 0) + 2 * cnt.get("FFMA2", 0)
        scalar = cnt.get("FADD", 0) + cnt.get("FMUL", 0) + 2 * cnt.get("FFMA", 0)
        per_pair = (2 * packed + scalar) / (2.0 * sources)
        res[kind] = max(res.get(kind, 0.0), per_pair)
    return res


if __name__ == "__main__":
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    print(p2p_flops_per_pair(sys.argv[1] if len(sys.argv) > 1 else
                             os.path.join(root, "paper_1106_5273_b200", "libfmm_b200.so")))


def sass_digest(lib, func_regex="k_p2p"):
    """sha1 of a kernel's SASS: ties an ncu flop count to the exact build."""
    import hashlib
    h = hashlib.sha1()
    for _, t in _sass(lib, func_regex):
        h.update(t.encode())
    return h.hexdigest()
