"""Census of the tensor-core / TMA / TMEM instructions in each kernel of the built library
(cuobjdump -sass), the static evidence that the kernels use tcgen05 (UTCHMMA), TMA
(UTMALDG), TMEM loads/stores (LDTM/STTM), commits (UTCBAR) and fp64 DMMA.

    python tools/sass_census.py [build_dir] > profiles/rNN/sass_census.txt
"""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "LDTM", "STTM", "DMMA", "ELECT", "SYNCS", "MUFU", "F2FP"]


def main(bdir):
    for obj in sorted(glob.glob(os.path.join(bdir, "*.cu.o"))):
        out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        fn, cnt = None, collections.OrderedDict()
        for line in out.splitlines():
            m = re.match(r"\s+Function : (\S+)", line)
            if m:
                fn = m.group(1)
                cnt[fn] = collections.Counter()
                continue
            if fn is None:
                continue
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", line)
            if m:
                op = m.group(1)
                if op in OPS:
                    cnt[fn][op] += 1
        for f, c in cnt.items():
            if any(c[o] for o in ("UTCHMMA", "UTCQMMA", "UTMALDG", "DMMA", "LDTM")):
                dem = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
                print(f"{os.path.basename(obj):22s} {dem[:100]}")
                print("    " + ", ".join(f"{o} {c[o]}" for o in OPS if c[o]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2503_18118_b200", "_build"))
