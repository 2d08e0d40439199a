mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -30 > gpurun_out/test.log
cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
cfg = fx.CONFIGS['C3']; arch = cfg.arch
m = ci.Model(arch, fx.make_weights(arch, 13), sys.argv[1] if len(sys.argv) > 1 else 'bf16')
n = 10240
x = torch.from_numpy(fx.make_inputs(arch, 1024, 10, 3).reshape(n, 3, 32, 32)).cuda()
h = torch.empty(n, 3072, device='cuda'); ws = m.workspace(1, n)
for _ in range(2): m.ci_forward_h(x, h, ws)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stage -s 3 -c 3 -o gpurun_out/prof_stage2 python /tmp/one.py > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
