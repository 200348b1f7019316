"""Symbolize SPQ_HOST_PROFILE samples: inclusive and exclusive time per function."""
import collections
import subprocess
import sys

lib = "paper_2010_06807_b200/libspaqr_b200.so"
lines = [l.split() for l in open(sys.argv[1]) if not l.startswith("#")]
addrs = sorted({a for l in lines for a in l if a != "?"})
# -a prints each address before its (possibly inlined) frames; keep the
# outermost function of the inline chain (the frame that really executes)
out = subprocess.run(["addr2line", "-a", "-f", "-C", "-i", "-e", lib] + ["0x" + a for a in addrs],
                     capture_output=True, text=True).stdout.splitlines()
name, cur, funcs = {}, None, []
def flush():
    if cur is not None:
        fn = [f for f in funcs if f and f != "??"]
        f = (fn[-1] if fn else "??").replace("(anonymous namespace)::", "")
        name[cur] = f.split("(")[0][:90] if not f.startswith("(") else f[:90]
k = 0
while k < len(out):
    ln = out[k]
    if ln.startswith("0x") and all(ch in "0123456789abcdefx" for ch in ln):
        flush()
        cur, funcs = ln[2:].lstrip("0") or "0", []
        k += 1
        continue
    funcs.append(ln)
    k += 2   # function line, then file:line
flush()
name = {a: name.get(a.lstrip("0") or "0", "??") for a in addrs}
excl, incl = collections.Counter(), collections.Counter()
n = len(lines)
for l in lines:
    fr = [name.get(a, "?") for a in l]
    # frame 0/1 are the handler / signal trampoline; first library frame = exclusive
    lib_frames = [f for f in fr if f != "?"]
    if fr and fr[0] != "?":
        excl[fr[0]] += 1
    elif lib_frames:
        excl["<outside lib> <- " + lib_frames[0]] += 1
    else:
        excl["<outside library>"] += 1
    for f in set(lib_frames):
        incl[f] += 1
print(f"{n} samples")
print("--- exclusive")
for f, c in excl.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{100 * c / n:6.1f}%  {f}")
print("--- inclusive")
for f, c in incl.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{100 * c / n:6.1f}%  {f}")
