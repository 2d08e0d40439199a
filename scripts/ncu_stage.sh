#!/bin/bash
# ncu --set full capture (with source) of one launch of stage S (0, 1, 2) of h on 10240 Arch-C images
# usage: scripts/ncu_stage.sh S NAME [bf16|fp32]
cd "$(dirname "$0")/.."
S=${1:-0}; NAME=${2:-stage}; PREC=${3:-bf16}
cat > /tmp/ncu_stage.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
arch = fx.CONFIGS['C3'].arch
m = ci.Model(arch, fx.make_weights(arch, 13), sys.argv[1])
n = 10240
x = torch.from_numpy(fx.make_inputs(arch, 1024, 10, 3).reshape(n, 3, 32, 32)).cuda()
h = torch.empty(n, 3072, device='cuda'); ws = m.workspace(1, n)
for _ in range(2):
    m.ci_forward_h(x, h, ws)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage -s $((3 + S)) -c 1 \
  -o gpurun_out/$NAME python /tmp/ncu_stage.py $PREC > gpurun_out/$NAME.log 2>&1
tail -3 gpurun_out/$NAME.log
