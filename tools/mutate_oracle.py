"""Mutation check of the oracle's pins: apply one plausible mistake at a time
to oracle/oracle.c, rebuild, run tests/test_oracle.py, and report whether a pin turned red.
usage: python tools/mutate_oracle.py [> profiles/r2_oracle_mutations.md]"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")

MUTATIONS = [
    ("G5 bin range lo = c-r+1", "lo[a] = o.c[a] - o.r;", "lo[a] = o.c[a] - o.r + 1;"),
    ("G5 bin range hi = c+r-2", "hi[a] = o.c[a] + o.r - 1;", "hi[a] = o.c[a] + o.r - 2;"),
    ("from_dense drops the last voxel", "for (uint64_t i = 0; i < n; ++i)\n    if (rgba[i])",
     "for (uint64_t i = 0; i + 1 < n; ++i)\n    if (rgba[i])"),
    ("rasteriser z range one short", "z < o.c[2] + o.r; ++z)", "z < o.c[2] + o.r - 1; ++z)"),
    ("slab_counts off by one in slab 0", "    out[z] = c;", "    out[z] = c + (z == 0);"),
    ("tmax inclusive (walk end)", "if (tcmp(&best, &te) >= 0) {", "if (tcmp(&best, &te) > 0) {"),
    ("clip strict (empty segment kept)", "if (tcmp(&ts, &te) >= 0) return 0;", "if (tcmp(&ts, &te) > 0) return 0;"),
    ("entry cell d>0 strict", "if (tcmp(&tm, &ts) <= 0) lo = mid;", "if (tcmp(&tm, &ts) < 0) lo = mid;"),
    ("entry cell d<0 strict", "if (tcmp(&tm, &ts) <= 0) hi = mid;", "if (tcmp(&tm, &ts) < 0) hi = mid;"),
    ("step sign ignored", "cell[a] += D[a] > 0 ? 1 : -1;", "cell[a] += 1;"),
    ("ties step one axis", "        last_axes |= 1 << a;\n      }", "        last_axes |= 1 << a;\n        break;\n      }"),
    ("zero-direction membership excludes o = 0", "if (O[a] < 0 || O[a] >=", "if (O[a] <= 0 || O[a] >="),
    ("t rounded at the wrong scale", "return (float)ldexpl(v, 14);", "return (float)ldexpl(v, 13);"),
    ("plane vs scalar compare scale", "l = (i128)a->N * ((i128)1 << 53);", "l = (i128)a->N * ((i128)1 << 52);"),
    ("entry face of the first cell dropped", "if (tcmp(&en, &ts) == 0) last_axes |= 1 << a;", "(void)en;"),
    ("normal sign flipped", "normal[3 * i + a] = rays[8 * i + 4 + a] > 0.0f ? -1 : 1;",
     "normal[3 * i + a] = rays[8 * i + 4 + a] > 0.0f ? 1 : -1;"),
    ("tmin rejected when negative", "(fabsf(tmin) >= 0x1p-16f && fabsf(tmin) < 0x1p20f)", "(tmin >= 0x1p-16f && tmin < 0x1p20f)"),
    ("plane time numerator sign", "int64_t N = P * ((int64_t)1 << 39) - O;", "int64_t N = P * ((int64_t)1 << 39) + O;"),
]


def main():
    orig = open(SRC).read()
    bak = SRC + ".bak"
    shutil.copy(SRC, bak)
    rows = []
    try:
        for name, old, new in MUTATIONS:
            assert orig.count(old) == 1, (name, orig.count(old))
            open(SRC, "w").write(orig.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle.py", "-x", "-q", "-p", "no:cacheprovider"],
                               cwd=ROOT, capture_output=True, text=True)
            failed = [l.split("::")[1].split(" ")[0] for l in r.stdout.splitlines() if l.startswith("FAILED")]
            rows.append((name, r.returncode != 0, failed[0] if failed else ""))
            print(f"{name}: {'killed' if r.returncode else 'SURVIVED'} {failed[:1]}", file=sys.stderr, flush=True)
    finally:
        shutil.copy(bak, SRC)
        os.remove(bak)
        subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=ROOT)
    print("# Oracle mutation check (tools/mutate_oracle.py)\n")
    print("One plausible mistake at a time in oracle/oracle.c; `tests/test_oracle.py -x` must turn red.\n")
    print("| mutation | result | first failing pin |\n|---|---|---|")
    for name, killed, t in rows:
        print(f"| {name} | {'killed' if killed else '**survived**'} | {t} |")
    print(f"\n{sum(k for _, k, _ in rows)} of {len(rows)} killed.")


if __name__ == "__main__":
    main()
