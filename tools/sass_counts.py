"""SASS evidence for profiles/: per sm_100a kernel of libgridse_b200.so, the counts of the instruction families the
design rests on -- FP64 tensor MMAs (DMMA), TMA bulk copies (UBLKCP), mbarrier operations (SYNCS), fences (MEMBAR),
FP atomics (none allowed: determinism) -- plus registers / spills from the cubin's resource usage.
    python tools/sass_counts.py > profiles/rNN_sass_counts.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_23175_b200", "libgridse_b200.so")
FAMILIES = [("DMMA", r"\bDMMA"), ("UBLKCP (TMA bulk)", r"\bUBLKCP"), ("SYNCS (mbarrier)", r"\bSYNCS"), ("LDGSTS (cp.async)", r"\bLDGSTS"),
            ("MEMBAR.*GPU", r"\bMEMBAR\.\w+\.GPU"), ("MEMBAR.*SYS", r"\bMEMBAR\.\w+\.SYS"), ("BAR", r"\bBAR\."),
            ("ATOM/RED integer", r"\b(ATOMG?|REDG?|RED)\.E\.(ADD|MAX|MIN)\.(?!F)"), ("ATOM/RED floating point", r"\b(ATOMG?|REDG?|RED)\.E\.\w+\.F(16|32|64)"),
            ("DFMA", r"\bDFMA"), ("DMUL", r"\bDMUL"), ("DADD", r"\bDADD"), ("MUFU.RSQ64H", r"MUFU\.RSQ64H"),
            ("LDG", r"\bLDG"), ("STG", r"\bSTG"), ("LDS", r"\bLDS"), ("STS", r"\bSTS"), ("SHFL", r"\bSHFL"),
            ("UTCMMA / LDTM (tcgen05; no FP64 kind exists)", r"\bUTC\w*MMA|\bLDTM"), ("STL/LDL (spill traffic)", r"\b(STL|LDL)\b")]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
usage = {}
for m in re.finditer(r"Function (\S+):\s*\n\s*(REG:\d+[^\n]*)", res):
    usage[m.group(1)] = m.group(2).strip()
kernels = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = kernels.setdefault(m.group(1), [])
        continue
    if cur is not None and re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
        cur.append(line)
arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
print(f"{os.path.relpath(LIB, ROOT)}: cubins for {', '.join(arch)}; {len(kernels)} kernels")
for name, body in kernels.items():
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    print(f"\n{dem[:150]}\n  instructions {len(body)}   {usage.get(name, '')}")
    text = "\n".join(body)
    row = [(lab, len(re.findall(pat, text))) for lab, pat in FAMILIES]
    print("  " + "   ".join(f"{lab} {n}" for lab, n in row if n or lab.startswith(("DMMA", "ATOM/RED floating", "UTCMMA"))))
