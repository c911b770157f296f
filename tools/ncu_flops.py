"""Hardware FP32 flops per launch from an ncu --metrics capture of the
sm__sass_thread_inst_executed_op_{fadd,fmul,ffma,fadd2,fmul2,ffma2}_pred_on
counters (thread-level instruction counts; a packed FP32x2 instruction carries
two lanes):  flops = fadd + fmul + 2 ffma + 2 (fadd2 + fmul2) + 4 ffma2.

  python tools/ncu_flops.py flops.csv [bench.json]    -> per-kernel table
With a bench JSON of the same command, the k_p2p row is written into
profiles/latest_p2p.json (hw_flops_ncu, pairs, SASS digest) for bench.py's
roofline."""
import collections
import csv
import json
import os
import sys

W = {"fadd": 1, "fmul": 1, "ffma": 2, "fadd2": 2, "fmul2": 2, "ffma2": 4}


def per_kernel(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    out = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("fmmb::<unnamed>::", "").replace("unnamed>::", "")
        d = out.setdefault((name, r[idi]), {"kernel": name, "flops": 0.0})
        m, v = r[mi], float(r[vi].replace(",", ""))
        if m == "gpu__time_duration.sum":
            d["ns"] = v
        for op, w in W.items():
            if m == "sm__sass_thread_inst_executed_op_%s_pred_on.sum" % op:
                d[op] = v
                d["flops"] += w * v
    for d in out.values():
        d["tflops"] = d["flops"] / d["ns"] / 1e3 if d.get("ns") else None
    return list(out.values())


if __name__ == "__main__":
    ks = per_kernel(sys.argv[1])
    for d in ks:
        print("%-24s %10.3f ms %14.4e flops %7.2f TFLOP/s" % (d["kernel"][:24], d["ns"] / 1e6, d["flops"], d["tflops"]))
    if len(sys.argv) > 2:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from tools.sass_flops import sass_digest
        b = json.loads([l for l in open(sys.argv[2]) if l.startswith("{")][-1])
        p2p = [d for d in ks if d["kernel"].startswith("k_p2p")][0]
        p = os.path.join(root, "profiles", "latest_p2p.json")
        prof = json.load(open(p)) if os.path.exists(p) else {}
        prof.update({"hw_flops_ncu": p2p["flops"], "hw_flops_ncu_pairs": b["p2p_pairs_per_step"],
                     "hw_flops_ncu_ms": p2p["ns"] / 1e6,
                     "hw_flops_ncu_counts": {k: p2p.get(k) for k in W},
                     "hw_flops_ncu_source": "ncu --metrics sm__sass_thread_inst_executed_op_*_pred_on, C3 bench, "
                                            "1 launch (%s)" % os.path.basename(sys.argv[1]),
                     "sass_sha1": sass_digest(os.path.join(root, "paper_1106_5273_b200", "libfmm_b200.so"))})
        json.dump(prof, open(p, "w"), indent=1)
        print("updated", p)
