"""Stall-reason breakdown (share of all samples) per hot-path stage of vd_device.cuh."""
import csv, re, subprocess, sys
from collections import defaultdict
from pathlib import Path

def main(rep):
    src = (Path(__file__).resolve().parents[1] / "paper_2509_12232_b200/csrc/vd_device.cuh").read_text().splitlines()
    marks = [(i + 1, m.group(1)) for i, l in enumerate(src) for m in [re.search(r"---- (A\d: \w+)", l)] if m]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f, hdr = None, None
    agg = defaultdict(lambda: defaultdict(float))
    for r in csv.reader(out.splitlines()):
        if len(r) == 2 and r[0] in ("File Name", "File Path"):
            f = r[1].rsplit("/", 1)[-1]; continue
        if r and r[0] == "Line No":
            hdr = r; continue
        if not (hdr and len(r) == len(hdr) and r[0]):
            continue
        ln = int(r[0]); key = f
        if f == "vd_device.cuh":
            key = "prologue"
            for s, name in marks:
                if ln >= s: key = name
        elif f.startswith("sm_100_rt"):
            key = "A3: intra"  # packed f32x2 intrinsics: the intra pair math
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                agg[key][h[6:]] += float(r[i] or 0)
    tot = sum(sum(d.values()) for d in agg.values())
    reasons = sorted({k for d in agg.values() for k in d}, key=lambda k: -sum(d[k] for d in agg.values()))[:9]
    print(f"{'stage':16s} {'all':>6s} " + " ".join(f"{k[:10]:>10s}" for k in reasons))
    for key, d in sorted(agg.items(), key=lambda x: -sum(x[1].values())):
        s = sum(d.values())
        print(f"{key[:16]:16s} {100*s/tot:5.1f}% " + " ".join(f"{100*d[k]/tot:9.1f}%" for k in reasons))

if __name__ == "__main__":
    main(sys.argv[1])
