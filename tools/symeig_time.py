import torch, time, sys
sys.path.insert(0, '.')
import paper_2206_15397_b200 as rk
for d in [int(a) for a in sys.argv[1:]] or [512, 2048, 4096]:
    g = torch.randn(d, min(d, 512), device='cuda')
    x = g @ g.T / g.shape[1] + 0.01 * torch.eye(d, device='cuda')
    x = 0.5 * (x + x.T)
    for _ in range(2):
        torch.cuda.synchronize(); t = time.time(); r = rk.sym_eig(x); torch.cuda.synchronize(); print(d, time.time() - t, flush=True)
