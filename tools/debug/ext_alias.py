"""Debug: torch.ops.sparrow.env_step with aliased mutable buffers (the C-ABI
rejects them with SP_EINVAL) -- does the error path work through the op?"""
import faulthandler
import os
import sys
faulthandler.enable()
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import torch  # noqa: E402
from helpers import config, load_maps, ranges  # noqa: E402
from paper_2305_04180_b200 import VecEnv, _lib  # noqa: E402
env = VecEnv(load_maps(1), 8, ranges(0.0), config(32))
env.reset_all(1)
ops = _lib.torch_ops()
D = env.state_dim
dev = env.device
a = torch.zeros(8, dtype=torch.int64, device=dev)
st = torch.empty((8, D), device=dev)
other = torch.empty((8, D), device=dev)
mk = lambda: (torch.empty(8, dtype=torch.float64, device=dev), torch.empty(8, dtype=torch.bool, device=dev),  # noqa: E731
              torch.empty(8, dtype=torch.bool, device=dev), torch.empty(8, dtype=torch.int8, device=dev))
r, dn, tr, ev = mk()
mode = sys.argv[1] if len(sys.argv) > 1 else "alias"
try:
    if mode == "alias":
        ops.env_step(env._h.value, a, st, st, r, dn, tr, ev)
    elif mode == "badaction":  # passes the op's checks; the kernel flags it lazily
        ops.env_step(env._h.value, a + 99, st, other, r, dn, tr, ev)
        env.check()
    elif mode == "shape":
        ops.env_step(env._h.value, a, st[:4], other[:4], r, dn, tr, ev)
    print(mode, "no error?!")
except Exception as e:  # noqa: BLE001
    print(mode, "raised", type(e).__name__, str(e)[:200])
