"""Aggregate an ncu source page (instructions, stall samples) by the phase
markers ('// ----' comments) of one kernel's source file."""
import csv
import io
import re
import subprocess
import sys


def main(rep, src_file, first_line, last_line):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    lines = open(src_file).read().splitlines()
    marks = [(i + 1, l.strip()[:60]) for i, l in enumerate(lines)
             if first_line <= i + 1 <= last_line and re.match(r"\s*// ----", l)]
    fname, hdr = "?", None
    agg = {}
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
            samp, inst = float(r[4]), float(r[7])
        except (ValueError, IndexError):
            continue
        ln = int(r[0])
        key = f"{fname} (helpers)"
        if fname == src_file.split("/")[-1] and first_line <= ln <= last_line:
            key = "preamble"
            for m, name in marks:
                if ln >= m:
                    key = f"{m}: {name}"
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += inst
        a[1] += samp
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% samp  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
