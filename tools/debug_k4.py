"""Debug helper: K4 on the GPU vs the reference golden for selected Gaussians."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests import golden_data as gd
from paper_2604_02586_b200.multiview import update_arrays, decompose_covariance
d = gd.load("scene21")
m = gd.motions(d)
dl, q, s, st = update_arrays(d["gaussians"], d["cameras"], m["status"], m["a"], m["b"],
                             m["weight_sum"], m["pixel_count"])
for i in (0, 7, 8):
    print(i, st[i], d["u_status"][i])
    print("  q  ", q[i], "\n  ref", d["u_rot"][i])
    print("  s  ", s[i], "\n  ref", d["u_scale"][i])
    print("  g q", d["gaussians"][i, 3:7])
fk = gd.load("fuse_kats")
bad = 0
for i in range(int(fk["n_dec"])):
    if int(fk[f"d{i}_st"]):
        qq, ss = decompose_covariance(fk[f"d{i}_sigma"], fk[f"d{i}_ref"], None)
        e = min(np.linalg.norm(qq - fk[f"d{i}_q"]), np.linalg.norm(qq + fk[f"d{i}_q"]))
        if e > 1e-7:
            bad += 1
            if bad < 3:
                print("dec", i, qq, fk[f"d{i}_q"], ss, fk[f"d{i}_s"])
print("decompose KAT bad", bad)
