"""Symbolize a SPQ_HOST_PROFILE dump (hostprof.cu) against the in-tree library.

    python tools/hostprof.py DUMP [top]

Prints inclusive sample counts per function (any frame) and the leaf
in-library function of each sample ("self"). Diagnostic only."""
import collections
import os
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2010_06807_b200", "libspaqr_b200.so")
lines = open(sys.argv[1]).read().splitlines()
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
samples = [l.split() for l in lines[1:]]
addrs = sorted({a for s in samples for a in s if a != "?"})
sym = {}   # address -> inlining chain, innermost first (addr2line -i)
if addrs:
    out = subprocess.run(["addr2line", "-a", "-f", "-C", "-i", "-e", LIB]
                         + [hex(int(a, 16) - 1) for a in addrs],
                         capture_output=True, text=True).stdout.splitlines()
    cur, i = None, 0
    while i < len(out):
        line = out[i]
        if line.startswith("0x"):
            cur = addrs[len(sym)]
            sym[cur] = []
            i += 1
            continue
        nm = line.replace("(anonymous namespace)::", "")
        sym[cur].append(nm.split("(")[0][:90])
        i += 2   # function, file:line


def ours(n):
    return not n.startswith(("std::", "__gnu_cxx", "void std::", "bool std::", "operator")) and n


incl, leaf, outside = collections.Counter(), collections.Counter(), collections.Counter()
for s in samples:
    names = [n for a in s if a != "?" for n in sym[a] if ours(n)]
    for n in set(names):
        incl[n] += 1
    if names:
        leaf[names[0]] += 1
        if s[0] == "?":
            outside[names[0]] += 1
print(f"{len(samples)} samples (250 us wall each)")
print("--- inclusive")
for n, c in incl.most_common(top):
    print(f"{c:7d} {100 * c / len(samples):5.1f}%  {n}")
print("--- leaf in-library frame (of which PC outside the library, e.g. CUDA driver / libc)")
for n, c in leaf.most_common(top):
    print(f"{c:7d} {outside[n]:7d}  {n}")
