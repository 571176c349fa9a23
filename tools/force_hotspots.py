"""k_force_reduce<false,false,false> hot spots by code region: executed warp instructions, stall
samples, lane efficiency, L1 shared wavefronts and global / local sectors, from an ncu source page
(SASS) and nvdisasm line info. Regions are marker-delimited line ranges of csrc/dem_kernels.cu and dem_math.cuh (ANCHORS).

usage: python tools/force_hotspots.py <ncu sass csv> <nvdisasm --print-line-info output>
"""
import collections
import csv
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_lines import line_map  # noqa: E402

SRC = __file__.rsplit("/", 2)[0] + "/paper_1503_03553_b200/csrc/"
# Regions as (file, start marker, end marker, name): each spans the lines from the first line
# containing its start marker up to (not including) the first later line containing its end
# marker, resolved against the current sources so the tool survives edits.
ANCHORS = [
    ("dem_kernels.cu", "__device__ __forceinline__ void integrate_particle(", "// the previous force kernel's pre-integrated",
     "pre-integration (next step's Integrate)"),
    ("dem_kernels.cu", "struct PairIdx {", "// The force kernel's shared-memory material table",
     "pair entries + partner / history prefetch"),
    ("dem_kernels.cu", "// The owner's previous history row entry", "// Pre-integration (single context",
     "history match"),
    ("dem_kernels.cu", "// Pre-integration (single context", "struct WarpMetrics {",
     "pre-integration (next step's Integrate)"),
    ("dem_kernels.cu", "// One contact of an owner (pi, vi, wi", "#ifndef DEM_FR_FAST",
     "contact body (partner state, table, memo)"),
    ("dem_kernels.cu", "#ifndef DEM_FR_FAST", "// The owner-major schedule of a unit",
     "FastMath flag / exact fallback"),
    ("dem_kernels.cu", "// The owner-major schedule of a unit", "__device__ __forceinline__ void force_reduce_tile(",
     "owner-major schedule"),
    ("dem_kernels.cu", "__device__ __forceinline__ void force_reduce_tile(", "// ---- B: lane = contact",
     "unit setup + phase A (owner staging)"),
    ("dem_kernels.cu", "// ---- B: lane = contact", "// ---- C: lane = owner",
     "phase B loop (gathers and owner state at chunk start, F/T and history stores)"),
    ("dem_kernels.cu", "// ---- C: lane = owner", "// metrics (pipeline.cpp:338-363)",
     "phase C (owner sums in list order)"),
    ("dem_kernels.cu", "// metrics (pipeline.cpp:338-363)", "// One contact of owner i with a history row",
     "tail (F, T out, metrics)"),
    ("dem_math.cuh", "struct V3 {", "// 256-bit global accesses", "math: vector ops"),
    ("dem_math.cuh", "// 256-bit global accesses", "// ---- fp64 divisions sharing one reciprocal",
     "256-bit loads / stores, x86 conversion"),
    ("dem_math.cuh", "// ---- fp64 divisions sharing one reciprocal", "struct MatPair {",
     "math: FastMath sqrt / reciprocal / division"),
    ("dem_math.cuh", "struct MatPair {", None, "math: geometry, coefficients, force, cap"),
]


def resolve():
    out = []
    for f, a, b, name in ANCHORS:
        lines = open(SRC + f).read().split("\n")
        start = next(k for k, l in enumerate(lines) if a in l) + 1
        end = len(lines) + 1 if b is None else next(k for k, l in enumerate(lines) if k + 1 > start and b in l) + 1
        out.append((f, start, end - 1, name))
    return out


K = resolve()


def region(loc):
    f, ln = loc
    for kf, a, b, name in K:
        if f == kf and a <= ln <= b:
            return name
    return "other: " + f


def main():
    csv_path, dis_path = sys.argv[1:3]
    dis = open(dis_path).read()
    fn = re.search(r"\.text\.(\S*k_force_reduceILb0ELb0ELb0E\S*)", dis).group(1)
    lm = line_map(dis_path, fn)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    col = {c: hdr.index(c) for c in ["Instructions Executed", "Thread Instructions Executed",
                                      "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared",
                                      "L2 Theoretical Sectors Global", "L2 Theoretical Sectors Local"]}
    body = [r for r in rows[2:] if r and r[0].startswith("0x")]
    base = int(body[0][0], 16)
    agg = collections.defaultdict(lambda: collections.Counter())
    for r in body:
        off = int(r[0], 16) - base
        loc, _ = lm.get(off, (("?", 0), ""))
        g = agg[region(loc)]
        for c, i in col.items():
            g[c] += int(float(r[i] or 0))
    tot = collections.Counter()
    for g in agg.values():
        tot.update(g)
    print("| region | warp insts % | stall samples % | lanes / inst | shared wavefronts % | global sectors % | local sectors |")
    print("|---|---|---|---|---|---|---|")
    for name, g in sorted(agg.items(), key=lambda kv: -kv[1]["Instructions Executed"]):
        e = g["Instructions Executed"]
        print(f"| {name} | {100 * e / tot['Instructions Executed']:.1f} | "
              f"{100 * g['Warp Stall Sampling (All Samples)'] / tot['Warp Stall Sampling (All Samples)']:.1f} | "
              f"{g['Thread Instructions Executed'] / max(e, 1):.1f} | "
              f"{100 * g['L1 Wavefronts Shared'] / max(tot['L1 Wavefronts Shared'], 1):.1f} | "
              f"{100 * g['L2 Theoretical Sectors Global'] / max(tot['L2 Theoretical Sectors Global'], 1):.1f} | "
              f"{g['L2 Theoretical Sectors Local']} |")
    print(f"\ntotals (all captured launches): {tot['Instructions Executed']:.4g} warp insts, "
          f"{tot['L1 Wavefronts Shared']:.4g} shared wavefronts, {tot['L2 Theoretical Sectors Global']:.4g} "
          f"global sectors, {tot['L2 Theoretical Sectors Local']:.4g} local sectors")


if __name__ == "__main__":
    main()
