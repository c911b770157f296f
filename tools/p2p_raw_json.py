"""Development tool: copy the k_p2p figures of an `ncu --set full` raw CSV
(`ncu -i rep --page raw --csv`) into profiles/latest_p2p.json (DRAM bytes per
launch, FMA-pipe / issue / warp utilisation, registers, SM clock), which
bench.py's roofline reads as `traffic` and `profile`.

  python tools/p2p_raw_json.py RAW.csv NOTE"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[0]
    d = dict(zip(h, rows[-1]))

    def f(k):
        return float(d[k].replace(",", ""))

    def unit(k):
        return dict(zip(h, rows[1])).get(k, "")

    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = f("dram__bytes_read.sum") * scale.get(unit("dram__bytes_read.sum"), 1)
    wr = f("dram__bytes_write.sum") * scale.get(unit("dram__bytes_write.sum"), 1)
    tu = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(
        unit("gpu__time_duration.sum"), 1e-6)
    p = os.path.join(ROOT, "profiles", "latest_p2p.json")
    prof = json.load(open(p)) if os.path.exists(p) else {}
    prof.update({
        "kernel": d["Kernel Name"][:80],
        "gpu_time_ms": f("gpu__time_duration.sum") * tu,
        "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
        "fma_pipe_active_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": int(f("launch__registers_per_thread")),
        "sm_clock_ghz": f("smsp__cycles_elapsed.avg.per_second") * {"Ghz": 1.0, "GHz": 1.0, "Mhz": 1e-3, "MHz": 1e-3,
                                                                    "cycle/nsecond": 1.0}.get(
            unit("smsp__cycles_elapsed.avg.per_second"), 1e-9),
        "source": "ncu --set full --clock-control none, C3 bench command, 1 launch (%s)" % os.path.basename(sys.argv[1]),
        "commit_note": sys.argv[2] if len(sys.argv) > 2 else "",
    })
    json.dump(prof, open(p, "w"), indent=1)
    print("updated", p, {k: prof[k] for k in ("gpu_time_ms", "dram_bytes_per_launch", "fma_pipe_active_pct")})


if __name__ == "__main__":
    main()
