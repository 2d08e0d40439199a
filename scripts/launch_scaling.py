"""Per-stage launch time of the fused stage kernel vs launch size (forward and inverse),
C3 arch, single stream: exposes fixed per-launch costs and wave quantisation."""
import sys, torch
sys.path.insert(0, '.')
import fixtures as fx
from paper_2106_06445_b200 import codedinv as ci
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
arch = fx.CONFIGS['C3'].arch
m = ci.Model(arch, fx.make_weights(arch, 13), prec)
xs = torch.from_numpy(fx.make_inputs(arch, 1024, 11, 3).reshape(11264, 3, 32, 32)).cuda()
for n in (148, 296, 1024, 2048, 4096, 10240, 11264):
    x = xs[:n].contiguous()
    h = torch.empty(n, 3072, device='cuda'); ws = m.workspace(1, n)
    for mode in ("fwd", "inv"):
        fn = (lambda: m.ci_forward_h(x, h, ws)) if mode == "fwd" else (lambda: m.ci_inverse_h(h, x, ws))
        fn(); torch.cuda.synchronize()
        ci.ci_test_prof_enable(True)
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        r = ci.ci_test_prof_read()
        ci.ci_test_prof_enable(False)
        ms = r[0] if isinstance(r, tuple) else r["ms"]
        print(mode, n, [round(v / 5, 4) for v in list(ms)[:3]], flush=True)
