"""Top stalled SASS instructions of one kernel by stall reason, with source lines.

usage: python tools/sass_stalls.py <ncu sass csv> <nvdisasm --print-line-info output> <mangled fn> [reason] [top]
reason: a column of the ncu source page (stall_long_sb, stall_wait, stall_short_sb, ...).
"""
import csv
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_lines import line_map  # noqa: E402


def main():
    csv_path, dis_path, fn = sys.argv[1:4]
    reason = sys.argv[4] if len(sys.argv) > 4 else "stall_long_sb"
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
    lm = line_map(dis_path, fn)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ir = hdr.index(reason)
    body = [r for r in rows[2:] if r and r[0].startswith("0x")]
    base = int(body[0][0], 16)
    tot = {h: 0 for h in hdr if h.startswith("stall_") and "Not Issued" not in h}
    for r in body:
        for h in tot:
            tot[h] += int(r[hdr.index(h)] or 0)
    allS = sum(tot.values())
    print("stall samples by reason:", ", ".join(f"{k[6:]} {100*v/allS:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
    items = sorted(body, key=lambda r: -int(r[ir] or 0))[:top]
    for r in items:
        off = int(r[0], 16) - base
        loc, _ = lm.get(off, (("?", 0), ""))
        print(f"{off:6x} {int(r[ir] or 0):6d} {loc[0]}:{loc[1]:<5} {r[1][:70]}")


if __name__ == "__main__":
    main()
