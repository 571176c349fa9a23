"""Per-source-line L1 traffic of one kernel: shared-memory wavefronts (and the excess from bank
conflicts) and global L1 tag requests / L2 sectors, from an ncu source page (SASS) + nvdisasm line info.

usage: python tools/sass_mem.py <ncu sass csv> <nvdisasm --print-line-info output> <mangled fn> [top]
"""
import collections
import csv
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_lines import line_map  # noqa: E402


def main():
    csv_path, dis_path, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    lm = line_map(dis_path, fn)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    cols = ["L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive", "L2 Theoretical Sectors Global",
            "L2 Theoretical Sectors Local", "L1 Tag Requests Global", "Instructions Executed"]
    idx = [hdr.index(c) for c in cols]
    body = [r for r in rows[2:] if r and r[0].startswith("0x")]
    base = int(body[0][0], 16)
    per = collections.defaultdict(lambda: [0] * len(cols))
    tot = [0] * len(cols)
    for r in body:
        off = int(r[0], 16) - base
        loc, _ = lm.get(off, (("?", 0), ""))
        for k, i in enumerate(idx):
            v = int(float(r[i] or 0))
            per[loc][k] += v
            tot[k] += v
    print("totals:", ", ".join(f"{c} {t:.4g}" for c, t in zip(cols, tot)))
    print("-- by shared wavefronts --")
    for loc, v in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{loc[0]}:{loc[1]:<5} shared wf {v[0]:>9} (excess {v[1]:>8})  insts {v[5]}")
    print("-- by global L2 sectors --")
    for loc, v in sorted(per.items(), key=lambda kv: -kv[1][2])[:top]:
        print(f"{loc[0]}:{loc[1]:<5} sectors {v[2]:>9} tag req {v[4]:>8} local {v[3]}  insts {v[5]}")


if __name__ == "__main__":
    main()
