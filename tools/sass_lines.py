"""Attribute ncu's per-SASS-instruction warp-stall samples to CUDA source lines.

    python tools/sass_lines.py REPORT.ncu-rep KERNEL_REGEX OBJ_OR_CUBIN [--top 40]

ncu's source page is read with --print-source sass; the same kernel is disassembled from the
object (nvdisasm -g, built with -lineinfo) and instructions are matched by position, so the object
must be the one that was profiled (the tool checks the instruction counts agree).
"""

import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile


def sass_samples(report, kernel):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "-k",
                          f"regex:{kernel}", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    # only the first kernel instance
    out_rows = []
    for r in rows:
        if r.get("Address", "").startswith("Address"):
            break
        out_rows.append(r)
    return out_rows


def cubin_of(path, tmp):
    if path.endswith(".cubin"):
        return path
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(path)], cwd=tmp, check=True,
                   capture_output=True)
    return os.path.join(tmp, next(f for f in os.listdir(tmp) if f.endswith(".cubin")))


def disasm_lines(cubin, kernel):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True,
                         check=True).stdout
    funcs = re.split(r"\n\s*\.text\.", txt)
    pat = re.compile(kernel)
    best = None
    for f in funcs:
        name = f.split(":", 1)[0].strip()
        if pat.search(name) and (best is None or len(f) > len(best[1])):
            best = (name, f)
    cur = ("?", 0)
    seq = []
    for ln in best[1].splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
            seq.append(cur)
    return best[0], seq


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("obj")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--sass-kernel", default=None,
                    help="regex on the mangled name for nvdisasm (default: KERNEL_REGEX)")
    a = ap.parse_args()
    rows = sass_samples(a.report, a.kernel)
    with tempfile.TemporaryDirectory() as tmp:
        name, seq = disasm_lines(cubin_of(a.obj, tmp), a.sass_kernel or a.kernel)
    print(f"kernel {name}: {len(rows)} profiled SASS instructions, {len(seq)} disassembled")
    if len(rows) != len(seq):
        print("WARNING: instruction counts differ; the object is not the profiled build")
    agg = collections.Counter()
    issued = collections.Counter()
    total = 0
    for r, loc in zip(rows, seq):
        s = int(r.get("Warp Stall Sampling (All Samples)", "0") or 0)
        agg[loc] += s
        issued[loc] += int(r.get("Instructions Executed", "0") or 0)
        total += s
    print(f"{'samples':>8} {'share':>6} {'warp-instr':>11}  file:line")
    for loc, s in agg.most_common(a.top):
        print(f"{s:>8} {100.0 * s / max(total, 1):>5.1f}% {issued[loc]:>11}  {loc[0]}:{loc[1]}")


if __name__ == "__main__":
    main()
