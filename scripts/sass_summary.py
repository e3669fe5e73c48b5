"""Per-kernel SASS instruction-class counts of libbl.so (cuobjdump -sass), the evidence of
which hardware paths each kernel uses: python scripts/sass_summary.py > profiles/r02_sass_summary.md"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1701_05936_b200/libbl.so"
CLASSES = [
    ("DMMA", r"\bDMMA\b"), ("IMMA", r"\bIMMA\b"), ("HMMA", r"\bHMMA\b"), ("UTCMMA (tcgen05)", r"\bUTC\w*MMA\b"),
    ("STTM (tcgen05.st)", r"\bSTTM"), ("LDTM (tcgen05.ld)", r"\bLDTM"), ("UTCBAR (tcgen05.commit)", r"\bUTCBAR"),
    ("UBLKCP (bulk copy)", r"\bUBLKCP\b"), ("UTMALDG (TMA)", r"\bUTMALDG\b"), ("SYNCS (mbarrier)", r"\bSYNCS\b"),
    ("STAS (st.async)", r"\bSTAS\b"), ("LDGSTS (cp.async)", r"\bLDGSTS\b"), ("DFMA", r"\bDFMA\b"),
    ("UCGABAR (cluster barrier)", r"\bUCGABAR"), ("LDG", r"\bLDG\b"), ("STG", r"\bSTG\b"),
    ("LDS", r"\bLDS\b"), ("SHFL", r"\bSHFL\b"), ("ATOMG/RED", r"\b(ATOMG|RED)\b"),
]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern and re.search(r"/\*[0-9a-f]{4,}\*/", line):
        for name, pat in CLASSES:
            if re.search(pat, line):
                counts[kern][name] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, r))


dm = demangle(list(counts))
print("# SASS instruction classes per kernel of libbl.so (sm_100a), round 2\n")
print("`cuobjdump -sass paper_1701_05936_b200/libbl.so`, counted by `scripts/sass_summary.py` (static instruction")
print("counts per kernel, not executed counts). Kernels of the hot path only; template instances summed by name.\n")
agg = collections.OrderedDict()
for k, c in counts.items():
    name = re.sub(r"\(.*", "", dm[k]).replace("void ", "").replace("bl::", "")
    base = re.sub(r"<.*", "", name)
    agg.setdefault(base, collections.Counter()).update(c)
cols = [c for c, _ in CLASSES]
print("| kernel | " + " | ".join(cols) + " |")
print("|---|" + "---|" * len(cols))
for base, c in agg.items():
    if not base.startswith("k_"):
        continue
    print(f"| `{base}` | " + " | ".join(str(c[x]) if c[x] else "" for x in cols) + " |")
tot = collections.Counter()
for c in agg.values():
    tot.update(c)
print("| **total** | " + " | ".join(str(tot[x]) for x in cols) + " |")
