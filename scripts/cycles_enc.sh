#!/bin/bash
# per-role cycle breakdown (CI_DEBUG_CYCLES) of the learned-encoder tail (E2, E3 on tcgen05), 1024 groups
cd "$(dirname "$0")/.."
PREC=${1:-fp32}
CI_DEBUG_PLAN=1 CI_DEBUG_CYCLES=1 timeout 120 python - "$PREC" <<'PY' 2>&1 | grep -E "cycles|plan"
import sys, torch
sys.path.insert(0, '.')
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
arch = fx.ARCH_CE
m = ci.Model(arch, fx.make_weights(arch, 14), sys.argv[1])
B, k = 1024, 2
x = torch.from_numpy(fx.make_inputs(arch, B, k, 4)).cuda()
xp = torch.empty(B, 3, 32, 32, device="cuda")
ws = m.workspace(k, B)
for _ in range(2):
    m.ci_encode(None, xp, ws, x=x, learned=True)
torch.cuda.synchronize()
PY
