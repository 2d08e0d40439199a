"""TMEM read bandwidth probe (ci_test_umma_rate variant 15), 148 CTAs, one per SM."""
import torch
from paper_2106_06445_b200 import codedinv as ci

iters = 4096
for nw in (4, 8, 16):
    for batch in (1, 2, 4):
        cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
        ci.ci_test_umma_rate(nw | (batch << 16) | (15 << 24), iters, 148, cyc)
        torch.cuda.synchronize()
        c = cyc.float().mean().item()
        print(f"[tmem ld] warps={nw:2d} loads/wait={batch}: {nw * iters * 2048 / c:6.1f} B/cycle/SM "
              f"({c / iters:.1f} cyc per warp-load round)")
