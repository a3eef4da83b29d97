"""Per-kernel SASS opcode summary of libqnn.so (cuobjdump -sass): the instructions that prove
the Blackwell-native path -- UTCIMMA (tcgen05.mma kind::i8), LDTM (tcgen05.ld), UTMALDG /
UTMASTG (TMA tensor load / store), UBLKCP (bulk copy) -- counted per kernel, plus spills
(LDL / STL) and the absence of legacy tensor instructions (HMMA / IMMA)."""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2006_10226_b200/libqnn.so"
OPS = ["UTCIMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "SYNCS", "LDL", "STL", "HMMA",
       "IMMA", "IDP"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
cnt = collections.defaultdict(collections.Counter)
fn = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and fn:
        op = m.group(1)
        cnt[fn]["_total"] += 1
        for o in OPS:
            if op == o:
                cnt[fn][o] += 1


def short(f):
    d = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
    return re.sub(r"\(.*", "", d)


fams = collections.defaultdict(lambda: collections.Counter())
nvar = collections.Counter()
for f, c in cnt.items():
    name = short(f)
    base = re.sub(r"<.*", "", name)
    nvar[base] += 1
    fams[base].update(c)
print(f"{'kernel family':44s} {'variants':>8s} " + " ".join(f"{o:>8s}" for o in OPS) + f" {'total':>9s}")
for base in sorted(fams):
    c = fams[base]
    print(f"{base[:44]:44s} {nvar[base]:8d} " + " ".join(f"{c[o]:8d}" for o in OPS) + f" {c['_total']:9d}")
