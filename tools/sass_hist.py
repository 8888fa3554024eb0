"""Per-kernel SASS instruction histograms of the built library objects
(Blackwell evidence: tcgen05 MMA / TMA / TMEM instructions).

  python tools/sass_hist.py > profiles/r02_sass_hist.txt

Counts every instruction (predicated ones included) per kernel function of
build/kernels/*.o and prints the Blackwell-specific mnemonics:
UTCHMMA/UTCQMMA (tcgen05.mma), UTCBAR (tcgen05.commit), LDTM/STTM (tcgen05.ld/st),
UTCATOMSWS (tcgen05.alloc/dealloc), UTMALDG/UTMASTG (TMA tensor loads/stores),
UBLKCP/UBLKPF (bulk copies / L2 prefetch), SYNCS (mbarrier), ELECT (elect.sync).
"""
import glob
import os
import re
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS", "UTMALDG", "UTMASTG", "UTMAPF", "UTMACCTL",
        "UBLKCP", "UBLKPF", "SYNCS", "ELECT", "HMMA"]
ins_re = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[0-9T]+\s+)?([A-Z][A-Z0-9_]*)")
fn_re = re.compile(r"Function : (\S+)")


def demangle(n):
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except OSError:
        return n


objs = sorted(glob.glob(os.path.join(ROOT, "paper_2101_07344_b200", "build", "kernels", "*.o")))
if not objs:
    sys.exit("no objects: run make -C paper_2101_07344_b200 first")
for o in objs:
    out = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
    per = defaultdict(Counter)
    fn = None
    for line in out.splitlines():
        m = fn_re.search(line)
        if m:
            fn = demangle(m.group(1))
            continue
        m = ins_re.search(line)
        if m and fn:
            per[fn][m.group(1)] += 1
    print(f"== {os.path.basename(o)}  (arch: {'sm_100a' if 'sm_100a' in out else '?'})")
    for f, c in sorted(per.items()):
        hits = {k: c[k] for k in KEYS if c[k]}
        if not hits:
            continue
        name = f.replace("(anonymous namespace)::", "").replace("void ", "")
        name = name[: name.find("(")] if "(" in name else name
        print(f"  {name}: total {sum(c.values())} | " + " ".join(f"{k}={v}" for k, v in hits.items()))
