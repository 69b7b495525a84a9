"""Dev: per-kernel SASS lines with the most stall samples / shared-memory excess wavefronts."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    lines = b.split("\n")
    name = lines[0][:80]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    iS, iSrc, iX, iW = h.index("# Samples"), h.index("Source"), h.index("L1 Wavefronts Shared Excessive"), h.index("L1 Wavefronts Shared")
    data = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(int(r[iS]) for r in data)
    print("==", name, "samples", tot, "excess smem wavefronts", sum(int(r[iX]) for r in data))
    for r in sorted(data, key=lambda r: -int(r[iS]))[:top]:
        print(f"  {int(r[iS]):6d} {r[iSrc].strip()[:70]:70s} xs={r[iX]} wf={r[iW]}")
    print("  -- top excess wavefronts")
    for r in sorted(data, key=lambda r: -int(r[iX]))[:6]:
        print(f"  {int(r[iS]):6d} {r[iSrc].strip()[:70]:70s} xs={r[iX]} wf={r[iW]}")
