"""Debug: forward h of Arch C images vs the oracle, per precision (run with/without CI_NO_STATIC)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import fixtures as fx
import oracle
from paper_2106_06445_b200 import codedinv as ci

arch = fx.ARCH_C
params = fx.make_weights(arch, 13)
n = 12
x = fx.make_inputs(arch, 1, n, 3)[0]
ref = oracle.forward_h(arch, params, x)
for prec in ("bf16", "fp32"):
    m = ci.Model(arch, params, prec)
    ws = m.workspace(1, n)
    h = torch.empty(n, arch.d, device="cuda")
    m.ci_forward_h(torch.from_numpy(x).cuda(), h, ws)
    torch.cuda.synchronize()
    e = np.max(np.abs(h.cpu().numpy() - ref), 1) / np.max(np.abs(ref), 1)
    print(os.environ.get("CI_NO_STATIC", "static"), prec, "max rel err", e.max())
