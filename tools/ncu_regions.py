"""Instruction / stall-sample shares per hot-path stage (line ranges of vd_device.cuh)."""
import re, sys
from collections import defaultdict
from pathlib import Path
sys.path.insert(0, str(Path(__file__).parent))
from ncu_lines import rows

def ranges():
    src = (Path(__file__).resolve().parents[1] / "paper_2509_12232_b200/csrc/vd_device.cuh").read_text().splitlines()
    marks = [(i + 1, m.group(1)) for i, l in enumerate(src) for m in [re.search(r"---- (A\d: \w+)", l)] if m]
    return marks

def main(rep):
    marks = ranges()
    agg = defaultdict(lambda: [0.0, 0.0])
    ti = ts = 0
    for f, ln, src, inst, samp in rows(rep):
        key = f
        if f == "vd_device.cuh":
            key = "vd_device.cuh:prologue"
            for start, name in marks:
                if ln >= start:
                    key = "vd_device.cuh:" + name
        agg[key][0] += inst
        agg[key][1] += samp
        ti += inst
        ts += samp
    for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:32s} inst {100*i/ti:5.1f}%  samples {100*s/ts:5.1f}%")

if __name__ == "__main__":
    main(sys.argv[1])
