"""Launch list of the learned encoder (ci_encode, CI_ENC_LEARNED) at k = 2, 4, 10 (run under ncu)."""
import sys, torch
sys.path.insert(0, '.')
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
arch = fx.ARCH_CE
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
m = ci.Model(arch, fx.make_weights(arch, 14), prec)
B = 1024
for k in (2, 4, 10):
    x = torch.from_numpy(fx.make_inputs(arch, B, k, 4)).cuda()
    xp = torch.empty(B, 3, 32, 32, device="cuda")
    ws = m.workspace(k, B)
    for _ in range(2):
        m.ci_encode(None, xp, ws, x=x, learned=True)
    torch.cuda.synchronize()
