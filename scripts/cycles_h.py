import sys, torch
sys.path.insert(0, ".")
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
arch = fx.CONFIGS["C3"].arch
m = ci.Model(arch, fx.make_weights(arch, 13), "fp32")
n = 10240
x = torch.from_numpy(fx.make_inputs(arch, 1024, 10, 3).reshape(n, 3, 32, 32)).cuda()
h = torch.empty(n, 3072, device="cuda"); ws = m.workspace(1, n)
m.ci_forward_h(x, h, ws); torch.cuda.synchronize()
