import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import torch, paper_2402_04396_b200 as q8p
art = open('/root/repo/tests/golden/e8p2_64x64.qshp','rb').read()
L = q8p.Layer.from_qshp(art, device=0)
x = torch.randn(1, 64, device='cuda')
y = L.forward(x); torch.cuda.synchronize(); print('ok', y.abs().sum().item())
