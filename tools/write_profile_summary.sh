#!/bin/bash
# Regenerate profiles/r01_ncu_full_summary.md and profiles/ncu_traffic.json from the
# captures tools/profile_all.sh leaves in gpurun_out/prof
set -e
cd /root/repo
P=gpurun_out/prof
{
  echo "# r01 ncu --set full summaries (B200, --clock-control none)"
  echo
  echo "Per-launch values from \`ncu -i <rep> --page raw\` (tools/ncu_summary.py); captured by"
  echo "tools/profile_all.sh. DRAM % is of ncu's theoretical peak; the bench roofline uses"
  echo "MEASURED_PEAKS.json instead. Absolute durations under ncu are cold-cache and serialised;"
  echo "compare shares, not absolutes, with the bench."
  echo
  echo "## config 1 (bench.py default: ada-PCG, SRHT, fp64, 2^16 x 1024) -- cfg1_full.ncu-rep"
  echo
  python tools/ncu_summary.py $P/cfg1_full.ncu-rep
  echo
  echo "## config 2 SJLT accumulation (bulk-copy streamed, fp64 2^20 x 2048, m = 2048) -- cfg2_sjlt_full.ncu-rep"
  echo
  python tools/ncu_summary.py $P/cfg2_sjlt_full.ncu-rep
  echo
  echo "## config 3 sketch kernel (TF32 tcgen05, m = 2048, n = 2^21, d = 4096) -- cfg3_tc_full.ncu-rep"
  echo
  python tools/ncu_summary.py $P/cfg3_tc_full.ncu-rep
  echo
  echo "SASS of k_gauss_tc: $(cuobjdump -sass build/adask/gauss_tc.o | grep -oE 'UTC[A-Z]*MMA[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|LDTM' | sort | uniq -c | tr '\n' ';' | tr -s ' ')"
  echo
  for M in 4096 32768; do
    echo "## config 4 block-SRHT (pipelined passes 1 / 2 + last-stage combine, fp32 2^21-row block, d = 1024, m = $M) -- cfg4_srht_m$M.ncu-rep"
    echo
    python tools/ncu_summary.py $P/cfg4_srht_m$M.ncu-rep
    echo
  done
  echo "SASS of the pipelined FWHT: $(cuobjdump -sass build/adask/srht_pipe.o | grep -oE 'UTMALDG[.A-Z0-9]*|UBLKCP[.A-Z0-9]*|FADD2' | sort | uniq -c | tr '\n' ';' | tr -s ' ')"
  echo "SASS of the SJLT accumulation: $(cuobjdump -sass build/adask/sjlt_pipe.o | grep -oE 'UBLKCP[.A-Z0-9]*|SYNCS[.A-Z0-9]*' | sort | uniq -c | tr '\n' ';' | tr -s ' ')"
} > profiles/r01_ncu_full_summary.md
python - <<'PY'
import csv, io, json, subprocess
def traffic(rep, pat):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out))); h = rows[0]
    tot = []
    for r in rows[2:]:
        if pat in r[h.index("Kernel Name")]:
            f = lambda k: float(r[h.index(k)].replace(",", "")) * (1e9 if "Gbyte" in rows[1][h.index(k)] else 1e6 if "Mbyte" in rows[1][h.index(k)] else 1e3 if "Kbyte" in rows[1][h.index(k)] else 1)
            tot.append(f("dram__bytes_read.sum") + f("dram__bytes_write.sum"))
    return tot
P = "gpurun_out/prof/"
t1 = traffic(P + "cfg1_full.ncu-rep", "k_hess_tma")
t4 = traffic(P + "cfg4_srht_m4096.ncu-rep", "k_")
t1s = traffic(P + "cfg1_full.ncu-rep", "k_fwht")  # pass 1, pass 2 of the first sketch, ...
out = {"cfg1": {"hess_mult": sum(t1) / len(t1), "srht": t1s[0] + t1s[1] if len(t1s) >= 2 else None},
       "cfg2": {"sjlt": sum(traffic(P + "cfg2_sjlt_full.ncu-rep", "k_sjlt_pipe"))},
       "cfg3": {"gaussian": sum(traffic(P + "cfg3_tc_full.ncu-rep", "k_gauss_tc"))},
       "cfg4": {"srht": sum(t4)},
       "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes) of the roofline unit, from "
               "profiles/r01_ncu_full_summary.md (cfg1: hess_mult mean, srht = both passes of the first sketch (m = 32); cfg2: SJLT accumulation m=2048; cfg3: TF32 "
               "sketch m=2048; cfg4: both SRHT passes + combine of one 2^21-row block at m=4096)"}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(out)
PY
cp gpurun_out/prof/cfg1_launches.csv profiles/r01_cfg1_launches.csv
echo wrote profiles/r01_ncu_full_summary.md
