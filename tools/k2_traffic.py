"""Write profiles/k2_traffic_<cfg>.json (per-launch DRAM bytes and executed warp instructions of
K2) from an `ncu --set full` report; bench.py reads it for roofline.traffic / issue_roofline.

    python tools/k2_traffic.py REPORT.ncu-rep cfg2 "profiles/r02_kernels_cfg2.txt (...)" [OUTDIR]
"""

import csv
import io
import json
import os
import subprocess
import sys


def main():
    rep, cfg, source = sys.argv[1], sys.argv[2], sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if "k2_raster" not in d.get("Kernel Name", ""):
            continue

        def val(m):
            return float(d[m].replace(",", "")) * scale.get(units.get(m, "byte"), 1.0)
        res = {"dram_bytes_per_launch": int(val("dram__bytes_read.sum") +
                                            val("dram__bytes_write.sum")),
               "executed_warp_instructions_per_launch":
                   int(float(d["smsp__inst_executed.sum"].replace(",", ""))),
               "source": source}
        outdir = sys.argv[4] if len(sys.argv) > 4 else os.path.join(
            os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
        path = os.path.join(outdir, f"k2_traffic_{cfg}.json")
        with open(path, "w") as f:
            json.dump(res, f)
        print(path, res)
        return
    sys.exit("no k2_raster launch in " + rep)


if __name__ == "__main__":
    main()
