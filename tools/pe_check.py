import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2505_11076_b200 as P
from paper_2505_11076_b200 import sharded
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = P.random_device_layer(8192, 8192, 8192, generator=g)
s = sharded.DeviceShard.from_device_layer(L, 0, 1, 0)
X = torch.randn((1, 8192), generator=g, device="cuda").half()
p = s.partial(X); q = s.partial_engine(X); torch.cuda.synchronize()
print("P diff", (p - q).abs().max().item(), p.abs().max().item(), q.abs().max().item())
yn = s.forward(X); ye = s.forward(X, engine=True); torch.cuda.synchronize()
print("y diff", (yn.float() - ye.float()).abs().max().item(), (yn != ye).sum().item(), yn.dtype, yn.abs().max().item())
