"""Dev: executed warp instructions by SASS opcode per kernel (ncu source page)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
for b in out.split('"Kernel Name"')[1:]:
    lines = b.split("\n")
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    iE, iSrc, iS = h.index("Instructions Executed"), h.index("Source"), h.index("# Samples")
    c = collections.Counter(); smp = collections.Counter()
    for r in rows[1:]:
        if len(r) != len(h): continue
        src = r[iSrc].strip()
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        op = op.split(".")[0]
        c[op] += int(r[iE] or 0); smp[op] += int(r[iS] or 0)
    tot = sum(c.values()); ts = sum(smp.values())
    print("==", lines[0][:90], f"total {tot:.3g} warp-instr")
    for op, v in c.most_common(18):
        print(f"  {op:10s} {v/tot*100:5.1f}%  samples {smp[op]/max(ts,1)*100:5.1f}%")
