"""Dump K4 intermediates (eigenvectors, eigenvalues, ref quat, covariance solution, quat) for
one Gaussian on the GPU."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from tests import golden_data as gd
from paper_2604_02586_b200 import _native as nat
lib = nat.lib()
lib.ts_debug_fuse_one.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(nat.Camera),
                                  ctypes.c_int32, ctypes.POINTER(nat.Motions),
                                  ctypes.POINTER(nat.Config), ctypes.c_int64, ctypes.c_void_p,
                                  ctypes.c_void_p]
d = gd.load("scene21")
m = gd.motions(d)
n, nv = len(d["gaussians"]), len(d["cameras"])
dev = "cuda"
g = torch.as_tensor(d["gaussians"], device=dev)
st = torch.as_tensor(m["status"].astype(np.int8).reshape(-1), device=dev)
a = torch.as_tensor(m["a"].reshape(-1, 4), device=dev)
b = torch.as_tensor(m["b"].reshape(-1, 2), device=dev)
w = torch.as_tensor(m["weight_sum"].reshape(-1), device=dev)
c = torch.as_tensor(m["pixel_count"].reshape(-1).astype(np.int32), device=dev)
mot = nat.Motions(st.data_ptr(), a.data_ptr(), b.data_ptr(), w.data_ptr(), c.data_ptr(), None, None)
cfg = nat.make_config()
np.set_printoptions(precision=10, linewidth=150)
for gi in (7, 8):
    dbg = torch.zeros(64, dtype=torch.float64, device=dev)
    nat.check(lib.ts_debug_fuse_one(g.data_ptr(), n, nat.make_cameras(d["cameras"]), nv,
                                    ctypes.byref(mot), ctypes.byref(cfg), gi, dbg.data_ptr(),
                                    nat.stream_ptr()))
    x = dbg.cpu().numpy()
    print(gi, "E", x[0:9], "\n ev", x[9:12], "\n ref", x[12:16], "\n sol", x[16:22], "\n q", x[22:26], "\n r", x[26:35], "\n best", x[35], "\n dots", x[36:45], "\n refm", x[45:54])
