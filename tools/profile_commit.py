"""Copy ncu evidence into profiles/ (tracked):

  full:      python tools/profile_commit.py full <rep.ncu-rep> <config> <kernel> <tag>
             -> profiles/<tag>_<config>_<kernel>.txt (metrics, stalls, hot lines) and the
                kernel's DRAM bytes per launch merged into profiles/<tag>_traffic.json
                (read by bench.py for roofline.traffic)
  launches:  python tools/profile_commit.py launches <launches.csv> <config> <tag>
             -> profiles/<tag>_<config>_launches.csv (+ per-kernel share summary .txt)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PDIR = os.environ.get("SPMMM_PROFILE_DIR", os.path.join(ROOT, "profiles"))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def full(rep, config, kernel, tag):
    import ncu_summary
    hdr, units, vals = ncu_summary.raw(rep)
    row = dict(zip(hdr, vals[0]))

    def num(k):
        try:
            return float(row[k].replace(",", ""))
        except (KeyError, ValueError):
            return None

    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
              "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    u = dict(zip(hdr, units))
    rd = num("dram__bytes_read.sum") * scale.get(u.get("dram__bytes_read.sum"), 1)
    wr = num("dram__bytes_write.sum") * scale.get(u.get("dram__bytes_write.sum"), 1)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep,
                            "25", "samp"], capture_output=True, text=True).stdout
    name = f"{tag}_{config}_{kernel}"
    with open(os.path.join(PDIR, name + ".txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on -k regex:{kernel} "
                f"-c 1 (config {config}); source report {os.path.basename(rep)}\n")
        f.write(out)
        f.write("\n# hottest source lines (share of warp instructions / stall samples)\n")
        f.write(lines)
    tpath = os.path.join(PDIR, f"{tag}_traffic.json")
    d = json.load(open(tpath)) if os.path.exists(tpath) else {
        "source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch",
        "configs": {}}
    d["configs"].setdefault(config, {})[kernel] = {
        "dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
        "duration_ms": num("gpu__time_duration.sum") * tscale.get(u.get("gpu__time_duration.sum"), 1.0),
        "report": name + ".txt"}
    json.dump(d, open(tpath, "w"), indent=1)
    print(f"wrote {name}.txt and {tag}_traffic.json ({(rd + wr) / 1e9:.3f} GB)")


def launches(csv_path, config, tag):
    text = open(csv_path).read()
    body = "\n".join(l for l in text.splitlines() if l.startswith('"'))
    rows = list(csv.DictReader(io.StringIO(body)))
    name = f"{tag}_{config}_launches"
    with open(os.path.join(PDIR, name + ".csv"), "w") as f:
        f.write(body + "\n")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        k = r["Kernel Name"].split("(")[0]
        tot[k] += float(r["Metric Value"])
        cnt[k] += 1
    all_ns = sum(tot.values())
    with open(os.path.join(PDIR, name + ".txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (config {config});\n"
                f"# cold-cache, serialised launches: compare SHARES, not absolute times\n")
        for k, ns in tot.most_common():
            f.write(f"{k:60s} launches {cnt[k]:4d}  avg {ns / cnt[k] / 1e3:10.1f} us  "
                    f"share {100 * ns / all_ns:5.1f}%\n")
    print(open(os.path.join(PDIR, name + ".txt")).read())


if __name__ == "__main__":
    os.makedirs(PDIR, exist_ok=True)
    if sys.argv[1] == "full":
        full(*sys.argv[2:6])
    else:
        launches(*sys.argv[2:5])
