"""profiles/ncu_traffic.json (the bench line's roofline.traffic) from the raw
pages of ncu --set full captures: DRAM bytes read + written per launch, averaged
over the launches of each kernel.
    python tools/ncu_traffic.py <tag> elasticity_q1_118=profiles/<tag>_loop_raw.csv.gz,profiles/<tag>_gnn_raw.csv.gz diffusion_fv_256=..."""
import csv
import gzip
import io
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TIME = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def rows_of(path):
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    return list(csv.reader(io.StringIO(f.read())))


def main():
    tag = sys.argv[1]
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    with open(out_path) as f:
        out = json.load(f)
    for arg in sys.argv[2:]:
        workload, paths = arg.split("=")
        for path in paths.split(","):
            rows = rows_of(path)
            hdr, units = rows[0], rows[1]
            ix = {h: i for i, h in enumerate(hdr)}
            acc = {}
            for r in rows[2:]:
                name = re.sub(r"^void\s+", "", r[ix["Kernel Name"]])
                name = name.replace("pclab_b200::", "").replace("<unnamed>::", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "")
                name = re.split(r"[<(]", name)[0]
                rd = float(r[ix["dram__bytes_read.sum"]]) * UNIT[units[ix["dram__bytes_read.sum"]]]
                wr = float(r[ix["dram__bytes_write.sum"]]) * UNIT[units[ix["dram__bytes_write.sum"]]]
                ms = float(r[ix["gpu__time_duration.sum"]]) * TIME[units[ix["gpu__time_duration.sum"]]]
                a = acc.setdefault(name, [0.0, 0.0, 0])
                a[0] += rd + wr
                a[1] += ms
                a[2] += 1
            for name, (b, ms, k) in acc.items():
                out.setdefault(workload, {})[name] = {
                    "dram_bytes": b / k, "ms_under_ncu": ms / k, "launches": k,
                    "source": f"ncu --set full --clock-control none ({os.path.relpath(path, ROOT)}, {tag}): "
                              "dram__bytes_read.sum + dram__bytes_write.sum per launch"}
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({w: {k: round(v["dram_bytes"] / 1e9, 3) for k, v in d.items()} for w, d in out.items()}, indent=1))


if __name__ == "__main__":
    main()
