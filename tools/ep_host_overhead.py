import time, torch, sys
sys.path.insert(0, '.')
from paper_2512_14080_b200 import ep, sonic
from paper_2512_14080_b200.inputs import make_expert_weights, make_token_inputs, CONFIGS
c = CONFIGS['7b']; T, d, n, E, K = c['T'], c['d'], c['n'], c['E'], c['K']
X, dO, S = make_token_inputs(T, d, E, seed=0, device='cuda')
W1, W2 = make_expert_weights(0, E, d, n, seed=0, device='cuda')
rk = ep.EPRank(T, d, n, E, K, 1, 0, W1, W2)
comm = ep.SimComm(1)
def step():
    ep.ep_forward([rk], comm, [X], [S]); ep.ep_backward([rk], comm, [dO])
for _ in range(3): step()
torch.cuda.synchronize()
N = 20
t0 = time.perf_counter(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
host = 0.0
for _ in range(N):
    h0 = time.perf_counter(); step(); host += time.perf_counter() - h0
e1.record(); torch.cuda.synchronize()
print(f"wall/step {(time.perf_counter()-t0)/N*1e3:.3f} ms  gpu/step {e0.elapsed_time(e1)/N:.3f} ms  host-issue/step {host/N*1e3:.3f} ms")
# pure issue cost of the fwd+bwd ops without GPU sync influence: time the python between syncs
