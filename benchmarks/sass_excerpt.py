#!/usr/bin/env python
"""SASS evidence for profiles/: instruction-class counts per kernel of libcbtm.so and the lines that
prove the mechanisms (256-bit loads, TMA bulk prefetch into L2 and programmatic dependent launch in
k_sum_reduce, TMA bulk stores in k_index_all, atomics / reductions and the fp64 classifier in the frame kernels).

    python benchmarks/sass_excerpt.py > profiles/r2b_sass_excerpt.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2407_02215_b200", "libcbtm.so")
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
kernels = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = []
        continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4,6}\*/", line):
        kernels[cur].append(line)
demangle = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
names = dict(zip(kernels, demangle))
CLASSES = ["UBLKCP", "UBLKPF", "SYNCS", "ACQBULK", "ATOMG", "ATOMS", "REDG", "RED.", "ATOM.", "DADD", "DMUL", "DFMA", "DSETP", "MUFU.RCP64H", "MUFU.RSQ64H",
           "POPC", "LOP3", "SHFL", "VOTE", "MATCH", "BAR.SYNC", "LDG.E.ENL2.256", "LDG", "STG", "LDS", "STS", "CCTL", "MEMBAR", "ERRBAR", "UTMALDG", "UTCHMMA", "HMMA"]


def mnemonic(line):
    m = re.search(r"\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    return m.group(1) if m else ""


print(f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)}: {len(kernels)} kernels (sm_100a)")
print("# instruction-class counts (static SASS), kernels with cbtm:: only\n")
for k, lines in kernels.items():
    nm = names.get(k, k)
    if "cbtm::" not in nm:
        continue
    ops = [mnemonic(l) for l in lines]
    counts = {c: sum(1 for o in ops if o.startswith(c)) for c in CLASSES}
    shown = ", ".join(f"{c.rstrip('.')} {n}" for c, n in counts.items() if n)
    no_return = sum(1 for l in lines if re.search(r"ATOMG\S* PT, RZ,", l))
    if no_return:
        shown += f" ({no_return} of the ATOMG write no result: destination RZ, fire and forget like REDG)"
    print(f"{nm.split('(')[0]}: {len(ops)} instructions; {shown}")

for want, pats in (("k_sum_reduce<true>", ("UBLKPF", "ACQBULK", "ATOM", "RED", "PREEXIT", "LDG", "POPC", "CCTL")),
                   ("k_index_all", ("UBLKCP", "FENCE", "DEPBAR", "LDG"))):
    for k, lines in kernels.items():
        if want in names.get(k, k):
            print(f"\n## {names[k].split('(')[0]}: loads, TMA bulk, dependent-launch, atomic and POPC instructions")
            for l in lines:
                if any(p in l for p in pats):
                    print("   " + l.strip()[:140])

# where the DFMAs of the frame kernel sit: only inside the expansions of __ddiv_rn / __dsqrt_rn / sin
for k, lines in kernels.items():
    nm = names.get(k, k)
    if "k_frames<2>" in nm:
        ops = [mnemonic(l) for l in lines]
        dfma = [i for i, o in enumerate(ops) if o.startswith("DFMA")]
        near = 0
        for i in dfma:
            window = ops[max(0, i - 40):i + 40]
            if any(o.startswith("MUFU.RCP64H") or o.startswith("MUFU.RSQ64H") for o in window):
                near += 1
        print(f"\n## {nm.split('(')[0]}: {len(dfma)} DFMA, {near} of them within 40 instructions of a MUFU.RCP64H / MUFU.RSQ64H "
              f"(the Newton steps of __ddiv_rn / __dsqrt_rn); the others belong to the slow paths of those expansions and to sin() "
              f"of the displacement demo.  The classifier's own products and sums are DMUL ({sum(1 for o in ops if o.startswith('DMUL'))}) "
              f"and DADD ({sum(1 for o in ops if o.startswith('DADD'))}): the library is built with -fmad=false and uses __dmul_rn / __dadd_rn.")
