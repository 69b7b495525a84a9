"""Dev: stall samples of a .ncu-rep kernel aggregated by SASS opcode, and the
sampled lines in program order with their share (coarse phase profile)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
for b in out.split('"Kernel Name"')[1:]:
    lines = b.split("\n")
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    iS, iSrc = h.index("# Samples"), h.index("Source")
    data = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(int(r[iS]) for r in data)
    agg = collections.Counter()
    for r in data:
        toks = r[iSrc].strip().split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        agg[op.split(".")[0]] += int(r[iS])
    print("==", lines[0][:70], "samples", tot)
    print("  by opcode:", ", ".join(f"{k} {v} ({100*v/tot:.0f}%)" for k, v in agg.most_common(14)))
    # program-order buckets of 64 instructions
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 80
    for i in range(0, len(data), B):
        s = sum(int(r[iS]) for r in data[i:i + B])
        if s * 50 >= tot:
            ops = collections.Counter(r[iSrc].strip().split()[0].split(".")[0] if not r[iSrc].strip().startswith("@") else r[iSrc].strip().split()[1].split(".")[0] for r in data[i:i + B])
            print(f"  [{i:5d}-{i+B:5d}] {s:6d} ({100*s/tot:4.1f}%)  " + " ".join(f"{k}:{v}" for k, v in ops.most_common(4)))
