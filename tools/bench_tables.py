"""Markdown tables of a profiling pass's bench lines (tools/run_profiles.sh output directory).

    python tools/bench_tables.py gpurun_out/r02
"""

import glob
import json
import os
import sys


def load(path):
    with open(path) as f:
        for ln in f:
            if ln.startswith("{"):
                return json.loads(ln)
    return None


def main():
    d = sys.argv[1]
    rows = []
    for cfg in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        b = load(os.path.join(d, f"bench_{cfg}.json"))
        if not b:
            continue
        e = b["e2e"]
        rf = b["roofline"]
        st = b["stage_ms"]
        seq = sum(st.values())
        rows.append(f"| {cfg} | {b['config']['n_gaussians'] // 1000}k x {b['config']['n_views']} x "
                    f"{b['config']['width']}x{b['config']['height']} | {b['ms_per_step']:.2f} "
                    f"({seq:.2f} seq.) | {b['value'] / 1e9:.2f} | {e['ms_per_step']:.2f} "
                    f"({e['zero_copy']['ms_per_step']:.2f} / {e['full_copy']['ms_per_step']:.2f}) | "
                    f"{e['value'] / 1e9:.2f} | {rf['kernel_ms']:.2f} | {rf['frac']:.3f} | "
                    f"{(rf['traffic'] or 0) / max(rf['algorithmic_bytes'], 1):.1f} |")
    print("| cfg | workload | ms/step resident | G GV/s | e2e ms headline (in place / whole copy) | e2e G GV/s "
          "| K2 ms | K2 HBM frac | K2 traffic / algorithmic |")
    print("|---|---|---|---|---|---|---|---|---|")
    print("\n".join(rows))
    print()
    print("| cfg | stage ms (K1 / depth sort / tile sort / K2 / K3 / K4) |")
    print("|---|---|")
    for cfg in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        b = load(os.path.join(d, f"bench_{cfg}.json"))
        if b:
            st = b["stage_ms"]
            print(f"| {cfg} | " + " / ".join(f"{v:.3f}" for v in st.values()) + " |")
    print()
    for name in ("bench_cfg5_clip8.json", "bench_cfg4_clip8.json", "bench_reference_cfg2.json"):
        b = load(os.path.join(d, name))
        if b:
            print(f"{name}: {b['ms_per_step']:.2f} ms/step, {b['value'] / 1e9:.4g} G GV/s, "
                  f"frames/s {b.get('frames_per_s')}, cpu {b.get('cpu_baseline', {}).get('sample')}")
    b = load(os.path.join(d, "bench_cfg2.json"))
    if b and b.get("cpu_baseline"):
        print("cfg2 cpu_baseline:", json.dumps(b["cpu_baseline"]))


if __name__ == "__main__":
    main()
