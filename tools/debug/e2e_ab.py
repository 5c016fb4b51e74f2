"""e2e host-buffer step: C-ABI sp_env_step_host vs torch copies + step_device (debug)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np, torch
from helpers import config, load_maps, ranges
from paper_2305_04180_b200 import VecEnv
from paper_2305_04180_b200.vecenv import StepBatch
n = 65536
env = VecEnv(load_maps(16), n, ranges(0.3), config(32), check_actions=False)
env.reset_all(0)
dev, D = env.device, env.state_dim
st = torch.cuda.current_stream()
acts = torch.randint(0, 5, (n,), dtype=torch.int64).pin_memory()
hb = env.host_buffers()
d_act = torch.empty(n, dtype=torch.int64, device=dev)
d_flat = torch.empty(hb.h_flat.numel(), dtype=torch.uint8, device=dev)
off = 0
views = []
for sh, dt, sz in ((n, torch.float64, 8), ((n, D), torch.float32, 4), ((n, D), torch.float32, 4),
                   (n, torch.bool, 1), (n, torch.bool, 1), (n, torch.int8, 1)):
    nb = int(np.prod(sh)) * sz
    views.append(d_flat[off:off + nb].view(dt).view(sh)); off += nb
r, s_, ss, dn, tr, ev = views
d_out = StepBatch(s_, r, dn, tr, ss, ev)
def c_path():
    env._lib.sp_env_step_host(env._h, acts.data_ptr(), hb.h_flat.data_ptr(), st.cuda_stream)
def torch_path():
    d_act.copy_(acts, non_blocking=True)
    env.step_device(d_act.data_ptr(), d_out)
    hb.h_flat.copy_(d_flat, non_blocking=True)
    st.synchronize()
for name, fn in (("c", c_path), ("torch", torch_path), ("c", c_path), ("torch", torch_path)):
    for _ in range(5): fn()
    ts = []
    for k in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); a.record(st); fn(); b.record(st); b.synchronize(); t1 = time.perf_counter()
        ts.append((a.elapsed_time(b), (t1 - t0) * 1e3))
    ev_ms = np.median([x for x, _ in ts]); wall = np.median([y for _, y in ts])
    print(f"{name:6s} events {ev_ms:.4f} ms  wall {wall:.4f} ms  -> {n / ev_ms * 1e3:.3e} env-steps/s")
