mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
cat > /tmp/cyc.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
prec = sys.argv[1]
cfg = fx.CONFIGS['C3']; arch = cfg.arch
m = ci.Model(arch, fx.make_weights(arch, 13), prec)
n = 10240
x = torch.from_numpy(fx.make_inputs(arch, 1024, 10, 3).reshape(n, 3, 32, 32)).cuda()
h = torch.empty(n, 3072, device='cuda'); ws = m.workspace(1, n)
m.ci_forward_h(x, h, ws); torch.cuda.synchronize()
import os; os.environ['CI_DEBUG_CYCLES'] = '1'
PY
CI_DEBUG_PLAN=1 timeout 120 python - bf16 <<'PY'
import os, sys
exec(open('/tmp/cyc.py').read())
PY
CI_DEBUG_PLAN=1 CI_DEBUG_CYCLES=1 timeout 120 python /tmp/cyc.py bf16 2>&1 | grep -E "cycles|plan"
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --no-alt --no-e2e --cpu-groups 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernels'], d['numerics'])"
