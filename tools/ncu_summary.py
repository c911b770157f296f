"""Summarise an ncu --csv launch list (per-kernel time, DRAM bytes and GB/s,
FMA-pipe and issue utilisation) into a JSON table for profiles/."""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launch = collections.OrderedDict()
    for r in rows[1:]:
        d = launch.setdefault(r[idi], {"name": r[ki].split("(")[0].replace("fmmb::<unnamed>::", "")
                                       .replace("void ", "")[:60]})
        try:
            d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        except ValueError:          # "n/a" (metric not collected for this launch)
            d[r[mi]] = 0.0
    agg = collections.OrderedDict()
    for d in launch.values():
        a = agg.setdefault(d["name"], collections.defaultdict(float))
        a["n"] += 1
        for k, v in d.items():
            if k != "name":
                a[k] += v
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        t = a["gpu__time_duration.sum"]
        b = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
        out.append(dict(kernel=k, launches=int(a["n"]), ms=t * 1e3, share=t / tot, dram_GB=b / 1e9,
                        dram_GBps=b / t / 1e9 if t > 0 else 0.0,
                        fma_pipe_pct=a.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 0) / a["n"],
                        issue_pct=a.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0) / a["n"],
                        tensor_pct=a.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                                         0) / a["n"]))
    return out, tot


if __name__ == "__main__":
    out, tot = summarise(sys.argv[1])
    print("%-60s %4s %9s %6s %8s %8s %6s %6s %6s" % ("kernel", "n", "ms", "share", "GB", "GB/s", "fma%", "issue%",
                                                     "tc%"))
    for r in out:
        print("%-60s %4d %9.3f %6.3f %8.3f %8.0f %6.1f %6.1f %6.1f" % (r["kernel"], r["launches"], r["ms"], r["share"],
                                                                      r["dram_GB"], r["dram_GBps"], r["fma_pipe_pct"],
                                                                      r["issue_pct"], r["tensor_pct"]))
    print("total ms %.3f" % (tot * 1e3))
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)
