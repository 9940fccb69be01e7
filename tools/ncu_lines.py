"""Per-source-line instruction counts and stall samples from an ncu report
(`--page source --print-source cuda,sass`); needs -lineinfo."""
import csv
import io
import subprocess
import sys


def main(rep, top=30, key="inst"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    fname = "?"
    hdr = None
    agg = []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            samp = float(r[4]); inst = float(r[7])
        except (ValueError, IndexError):
            continue
        agg.append((inst, samp, f"{fname}:{r[0]}", r[1].strip()[:90]))
    ti = sum(a[0] for a in agg) or 1
    ts = sum(a[1] for a in agg) or 1
    idx = 0 if key == "inst" else 1
    print(f"total warp-inst {ti:.3e}, stall samples {ts:.0f}")
    for inst, samp, loc, src in sorted(agg, key=lambda a: -a[idx])[:top]:
        print(f"{100*inst/ti:5.1f}% inst {100*samp/ts:5.1f}% samp  {loc:18s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30,
         sys.argv[3] if len(sys.argv) > 3 else "inst")
