"""Writes profiles/traffic.json from ncu --set full captures: DRAM bytes per launch of the named kernels, with the
commit the capture was taken at.  bench.py reads it for roofline.traffic (null when a kernel/config has no capture).

    python tools/ncu_traffic.py <config> <report.ncu-rep> [<config> <report> ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    args = sys.argv[1:]
    commit = os.environ.get("PM_COMMIT") or subprocess.run(["git", "-C", REPO, "rev-parse", "--short", "HEAD"],
                                                           capture_output=True, text=True).stdout.strip()
    path = os.path.join(REPO, os.environ.get("PM_PROFILES_DST", "profiles"), "traffic.json")
    rec = {"captures": []}
    if os.path.exists(path):
        rec = json.load(open(path))
    for config, rep in zip(args[::2], args[1::2]):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for v in rows[2:]:
            name = v[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0].strip()

            def val(metric):
                i = hdr.index(metric)
                x = float(v[i].replace(",", ""))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
                return x * scale
            entry = {"kernel": name, "config": config, "report": os.path.basename(rep), "commit": commit,
                     "dram_bytes_per_launch": int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum")),
                     "duration_us": float(v[hdr.index("gpu__time_duration.sum")].replace(",", "")) *
                     {"ns": 1e-3, "us": 1, "ms": 1e3, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(units[hdr.index("gpu__time_duration.sum")], 1)}
            rec["captures"] = [c for c in rec["captures"] if not (c["kernel"] == name and c["config"] == config)] + [entry]
            print(entry)
    json.dump(rec, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
