"""Instruction-level digest of an ncu report (source page, SASS): samples and executions per
opcode and the hottest instructions with their top stall reasons.

    python tools/ncu_hot.py REPORT.ncu-rep [N]
"""
import csv, sys, subprocess, collections
path = sys.argv[1]
out = subprocess.run(["ncu","-i",path,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iSrc = hdr.index("Source"); iE = hdr.index("Instructions Executed")
stall_cols = [i for i,h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iS] or 0) for r in data)
print("total samples", tot)
# opcode histogram weighted by samples and by executions
byop = collections.Counter(); byex = collections.Counter()
for r in data:
    op = r[iSrc].split()[0] if r[iSrc].split() else "?"
    if op.startswith("@"): op = r[iSrc].split()[1]
    op = op.split(".")[0]
    byop[op] += float(r[iS] or 0); byex[op] += float(r[iE] or 0)
totex = sum(byex.values())
print("by opcode (samples%, exec%)")
for op, v in byop.most_common(25): print(f"  {op:12s} {100*v/tot:6.2f}%  {100*byex[op]/totex:6.2f}%")
# top instructions
print("top instructions")
top = sorted(data, key=lambda r: -float(r[iS] or 0))[:int(sys.argv[2]) if len(sys.argv)>2 else 30]
for r in top:
    st = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:3]
    print(f"{r[0][-5:]} {float(r[iS])/tot*100:5.2f}% {r[iSrc].strip()[:60]:60s} " + " ".join(f"{n[6:]}={v:.0f}" for v,n in st))
