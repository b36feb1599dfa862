"""Single-process PeerComm smoke (virtual ranks on one GPU) with a watchdog traceback dump."""
import faulthandler
import sys
import time

import torch

sys.path.insert(0, ".")
faulthandler.dump_traceback_later(60, exit=True)
from paper_2512_14080_b200 import ep, sonic  # noqa: E402
from paper_2512_14080_b200.inputs import make_inputs  # noqa: E402

G, T, d, n, E, K = 2, 768, 128, 64, 16, 4
L = E // G
base = make_inputs(T, d, n, E, K, seed=40, device="cuda")
ins = [make_inputs(T, d, n, E, K, seed=41 + r, device="cuda") for r in range(G)]
ranks = [ep.EPRank(T, d, n, E, K, G, r, base.W1[r * L:(r + 1) * L].contiguous(),
                   base.W2[r * L:(r + 1) * L].contiguous()) for r in range(G)]
comm = ep.PeerComm(G, T, d, L, range(G))
print("created", flush=True)
for rk in ranks:
    print("stream", comm.streams, flush=True)
disp = []
for i, r in enumerate(ranks):
    with comm.rank_stream(i):
        disp.append(r.plan_fwd(ins[i].S))
print("planned", flush=True)
sc, rc = comm.exchange_counts_dev([c for _, c in disp])
print("counts", sc, rc, flush=True)
t0 = time.time()
Os = ep.ep_forward(ranks, comm, [i.X for i in ins], [i.S for i in ins])
torch.cuda.synchronize()
print("fwd ok", time.time() - t0, flush=True)
outs = ep.ep_backward(ranks, comm, [i.dO for i in ins])
torch.cuda.synchronize()
print("bwd ok", flush=True)
comm.close()
