import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np, torch
import oracle
from oracle import recurrent as OR
import paper_2502_15349_b200 as af
from paper_2502_15349_b200 import spec as S
from probe_linear import dev, rounded
sp = S.builtin("mamba2-ssm", batch=1, heads=1, seq=256, d_qk=128, d_v=128)
a = oracle.generate(sp, 5); d = dev(a)
dout = torch.tensor(np.random.default_rng(1).uniform(-1, 1, (1, 1, 256, 128)), device="cuda").bfloat16()
g = af.linear_backward(sp, d, dout)
gate, dec = d["gate"][..., 0].double(), d["decay"][..., 0].double()
dloga_k = (g["decay"][..., 0].double() * dec)
dq, dk = g["q"].double(), g["k"].double()
q, k = d["q"].double(), d["k"].double()
dq_dot = (q * dq).sum(-1)
dkm = dk / gate[..., None]
dk_dot = (k * dkm).sum(-1)
val = dq_dot - gate * dk_dot
dloga_t = torch.flip(torch.cumsum(torch.flip(val, [-1]), -1), [-1])
print("dloga kernel vs torch-from-outputs:", ((dloga_k - dloga_t).norm() / dloga_t.norm()).item())
print(dloga_k[0, 0, :8].cpu().numpy()); print(dloga_t[0, 0, :8].cpu().numpy())
print(dloga_k[0, 0, -8:].cpu().numpy()); print(dloga_t[0, 0, -8:].cpu().numpy())
gw = OR.chunk_vjp(sp, rounded(a), dout.double().cpu().numpy(), chunk=64)
print("oracle dloga", (gw["decay"][0, 0, :8, 0] * a["decay"][0, 0, :8, 0]))
