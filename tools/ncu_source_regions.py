"""Development tool: summarise an `ncu --page source --csv --print-source sass`
export of k_p2p -- warp-stall samples and executed warp instructions per code
region (SASS offset ranges of the far loop, the near loop, the rest), and the
instructions with the most not-issued samples.  Not part of the product path.

usage: python tools/ncu_source_regions.py SOURCE_SASS.csv FAR_LO FAR_HI NEAR_LO NEAR_HI [TOP]
(offsets in hex, from `cuobjdump -sass -fun <k_p2p>` of the same library)
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    far = (int(sys.argv[2], 16), int(sys.argv[3], 16))
    near = (int(sys.argv[4], 16), int(sys.argv[5], 16))
    top = int(sys.argv[6]) if len(sys.argv) > 6 else 15
    rows = [x for x in list(csv.reader(open(path)))[2:] if x and x[0].startswith("0x")]
    base = int(rows[0][0], 16)
    rec = [(int(x[0], 16) - base, x[1].strip(), int(x[2]), int(x[3]), int(x[5])) for x in rows]
    tot = sum(r[2] for r in rec) or 1
    totn = sum(r[3] for r in rec) or 1
    toti = sum(r[4] for r in rec) or 1

    def region(o):
        if far[0] <= o < far[1]:
            return "far loop"
        if near[0] <= o < near[1]:
            return "near loop (+close series)"
        return "staging/flush/other"

    acc = defaultdict(lambda: [0, 0, 0])
    for o, _, a, n, ie in rec:
        v = acc[region(o)]
        v[0] += a
        v[1] += n
        v[2] += ie
    print("%-28s %9s %11s %11s" % ("region", "samples", "not-issued", "warp-instr"))
    for k, v in sorted(acc.items()):
        print("%-28s %8.1f%% %10.1f%% %10.1f%%" % (k, 100 * v[0] / tot, 100 * v[1] / totn, 100 * v[2] / toti))
    print("\ntop %d instructions by not-issued samples (share of all not-issued samples):" % top)
    for o, s, a, n, ie in sorted(rec, key=lambda r: -r[3])[:top]:
        print("  %-7s %-22s %-58s %5.2f%%" % (hex(o), region(o), s[:58], 100 * n / totn))


if __name__ == "__main__":
    main()
