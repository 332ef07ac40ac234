"""Aggregate an ncu report's source page by CUDA source line:
instructions executed and warp-stall samples (development helper)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
tot_i = tot_s = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or r[0] in ("", "Function Name", "Kernel Name"):
        continue
    try:
        ins = int(r[hdr["Instructions Executed"]])
        smp = int(r[hdr["Warp Stall Sampling (All Samples)"]])
    except (ValueError, KeyError, IndexError):
        continue
    key = (fname, int(r[0]))
    agg[key][0] += ins
    agg[key][1] += smp
    agg[key][2] = r[1][:90]
    tot_i += ins
    tot_s += smp
print(f"total instructions {tot_i:.3e}  stall samples {tot_s}")
by_file = collections.defaultdict(lambda: [0, 0])
for (f, l), (i, s, _) in agg.items():
    by_file[f][0] += i
    by_file[f][1] += s
for f, (i, s) in sorted(by_file.items(), key=lambda kv: -kv[1][1]):
    print(f"  {f:14s} inst {100*i/tot_i:5.1f}%  samples {100*s/tot_s:5.1f}%")
key = 1 if (len(sys.argv) < 4 or sys.argv[3] == "samples") else 0
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{f:12s}:{l:<5d} inst {100*i/tot_i:5.2f}%  samp {100*s/tot_s:5.2f}%  {src.strip()}")
