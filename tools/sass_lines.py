"""Per-source-line hot spots of one kernel from an ncu SASS page + nvdisasm line info.

usage: python tools/sass_lines.py <ncu sass csv> <nvdisasm --print-line-info output> <mangled fn> [top]

The ncu CSV comes from `ncu -i rep --page source --csv --kernel-name regex:K --print-source sass`;
addresses are matched by offset from the function start. Prints the top source lines by
executed warp instructions and by stall samples.
"""
import collections
import csv
import re
import sys


def line_map(dis_path, fn):
    out, cur, inside = {}, None, False
    hdr = re.compile(r'//## File "([^"]+)", line (\d+)')
    ins = re.compile(r'/\*([0-9a-f]{4,})\*/\s+(.*?);')
    for raw in open(dis_path):
        if raw.startswith("//---------------------"):
            inside = (".text." + fn + " ") in raw
            continue
        if not inside:
            continue
        m = hdr.search(raw)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = ins.search(raw)
        if m:
            out[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return out


def main():
    csv_path, dis_path, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    lm = line_map(dis_path, fn)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ia = hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    ithr = hdr.index("Thread Instructions Executed")
    body = [r for r in rows[2:] if r and r[0].startswith("0x")]
    base = int(body[0][0], 16)
    per_line = collections.defaultdict(lambda: [0, 0, 0])
    per_op = collections.Counter()
    tot = [0, 0, 0]
    for r in body:
        off = int(r[0], 16) - base
        loc, _ = lm.get(off, (("?", 0), ""))
        e, s, t = int(r[ia] or 0), int(r[isamp] or 0), int(r[ithr] or 0)
        per_line[loc][0] += e
        per_line[loc][1] += s
        per_line[loc][2] += t
        toks = [t for t in r[1].split() if not t.startswith("@")]
        per_op[toks[0].split(".")[0] if toks else "?"] += e
        tot[0] += e; tot[1] += s; tot[2] += t
    print(f"total warp insts {tot[0]:.4g}  samples {tot[1]}  thread insts/warp inst {tot[2]/max(tot[0],1):.1f}")
    print("-- by executed warp instructions --")
    for loc, v in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{loc[0]}:{loc[1]:<5} insts {v[0]:>10} ({100*v[0]/tot[0]:5.1f}%)  samples {100*v[1]/max(tot[1],1):5.1f}%  thr/inst {v[2]/max(v[0],1):5.1f}")
    print("-- by stall samples --")
    for loc, v in sorted(per_line.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{loc[0]}:{loc[1]:<5} samples {100*v[1]/max(tot[1],1):5.1f}%  insts {100*v[0]/tot[0]:5.1f}%")
    print("-- opcodes by executed warp instructions --")
    for op, n in per_op.most_common(25):
        print(f"{op:10s} {n:>10} {100*n/tot[0]:5.1f}%")


if __name__ == "__main__":
    main()
