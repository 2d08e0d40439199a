"""Debug: one coupling block with Arch C stage-1 shape (C=48, 8x8, c=24, m=128) vs the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import fixtures as fx
import oracle
from paper_2106_06445_b200 import codedinv as ci

arch = fx.Arch("S1", 48, 8, 8, (fx.Stage(0, 1, 128),), heads=())
params = fx.make_weights(arch, 3)
n = 22
x = (np.random.default_rng(0).random((n, 48, 8, 8))).astype(np.float32)
ref = oracle.forward_h(arch, params, x).reshape(n, 48, 64)
for prec in ("bf16",):
    m = ci.Model(arch, params, prec)
    ws = m.workspace(1, n)
    h = torch.empty(n, arch.d, device="cuda")
    m.ci_forward_h(torch.from_numpy(x).cuda(), h, ws)
    torch.cuda.synchronize()
    g = h.cpu().numpy().reshape(n, 48, 64)
    err = np.abs(g - ref).max(axis=(0, 2))
    print(os.environ.get("CI_NO_STATIC", "static"), prec, "per-channel max abs err:")
    print(np.array2string(err, precision=3, max_line_width=200))
    d = (g - ref)[0, 24:48]
    print("img0 ch24.. err at pixel 0..7:", np.array2string(d[:, :4], precision=3, max_line_width=200))
    # is output channel o equal to ref channel o' for some permutation?
    for o in range(24, 48):
        best = min(range(24, 48), key=lambda q: np.abs(g[:, o] - ref[:, q]).max())
        if best != o: print("ch", o, "matches ref ch", best, np.abs(g[:, o] - ref[:, best]).max())
