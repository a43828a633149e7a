"""Per-source-line instruction / stall-sample totals from an ncu report (--import-source)."""
import csv, subprocess, sys
from collections import defaultdict

def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f = None
    hdr = None
    for r in csv.reader(out.splitlines()):
        if len(r) == 2 and r[0] == "File Path":
            f = r[1].rsplit("/", 1)[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            yield f, int(r[0]), r[1], float(r[7] or 0), float(r[4] or 0)

def main(rep, top=40):
    agg = []
    ti = ts = 0
    for f, ln, src, inst, samp in rows(rep):
        agg.append((inst, samp, f, ln, src))
        ti += inst; ts += samp
    agg.sort(reverse=True)
    print(f"total warp-inst {ti:.4g}, samples {ts:.4g}")
    for inst, samp, f, ln, src in agg[:int(top)]:
        print(f"{100*inst/ti:5.1f}% inst {100*samp/ts:5.1f}% samp  {f}:{ln}  {src.strip()[:90]}")
    return agg

if __name__ == "__main__":
    main(*sys.argv[1:])
