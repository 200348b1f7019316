"""Leaf runtime.cu line histogram of a SPQ_HOST_PROFILE dump (run on the box that built the profiled library). Diagnostic only."""
import collections, subprocess, sys
import os
LIB=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),"paper_2010_06807_b200","libspaqr_b200.so")
lines=open(sys.argv[1]).read().splitlines()
samples=[l.split() for l in lines[1:]]
addrs=sorted({a for s in samples for a in s if a!="?"})
out=subprocess.run(["addr2line","-a","-f","-C","-i","-e",LIB]+[hex(int(a,16)-1) for a in addrs],capture_output=True,text=True).stdout.splitlines()
sym={};cur=None;i=0
while i<len(out):
    l=out[i]
    if l.startswith("0x"):
        cur=addrs[len(sym)];sym[cur]=[];i+=1;continue
    sym[cur].append((l.split("(")[0][:60],out[i+1].split("/")[-1]));i+=2
cnt=collections.Counter()
for s in samples:
    # first frame whose file is runtime.cu
    done=False
    for a in s:
        if a=="?":continue
        for fn,fl in sym[a]:
            if fl.startswith("runtime.cu"):
                cnt[(fn,fl)]+=1;done=True;break
        if done:break
for (fn,fl),c in cnt.most_common(70):
    print(c,fn,fl)
