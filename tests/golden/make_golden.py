"""Regenerate tests/golden/* from the UNMODIFIED reference (run in the build
container, where /root/reference and oracle/_ref exist):

    ./oracle/build_ref.sh && python tests/golden/make_golden.py

Outputs (committed; the GPU box has no /root/reference):
* maps16.npz      -- ``generate_maps(16, seed=0, size_cm=366, density=0.08)``
  (mapgen.py:111-115, the ``color mapgen`` defaults, cli.py:54-56) saved as
  text and re-loaded with ``GridMap.from_text`` exactly as the reference CLI
  consumes maps; packed occupancy + goal/spawn + sha256 of each text.
* traj_cfg1.npz   -- cfg1: 16 envs, map00, 32 beams, default DiversityRanges,
  Philox random actions, 1000 steps, run by the reference VecEnv with its
  per-lane numpy streams replaced by the Philox contract
  (oracle/philox_shim.py).  Rewards/events/dones full; obs every 50 steps.
* traj_cfg2.npz   -- cfg2 slice: 256 envs over the 16 maps, diversity 0.3,
  32 beams, 100 steps (same recording).
* rays16.npz      -- kernels.cast_rays (Cython backend) on 16 maps x 3 max
  ranges x 512 random free poses (x, y, heading stored) x 32 beams, the
  directions built as core.py:223-232 does; disc_collides on the same poses.
* replay.npz      -- ReplayBuffer.sample indices/rows under a Philox stream.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
OUT = os.path.dirname(os.path.abspath(__file__))

from oracle import oracle as O  # noqa: E402
from oracle.philox_shim import PhiloxStream, random_actions, reference_rng_proxy  # noqa: E402

R = 32


def save_maps(maps_text):
    from color_rl.sim.gridmap import GridMap
    occ, meta, shas = [], [], []
    for t in maps_text:
        m = GridMap.from_text(t)
        occ.append(np.packbits(m.occupancy, axis=1))
        meta.append([*m.goal_center, m.goal_radius_cm, *m.spawn_region, m.width_cm, m.height_cm,
                     m.cell_size_cm])
        shas.append(hashlib.sha256(t.encode()).hexdigest())
    np.savez_compressed(os.path.join(OUT, "maps16.npz"), occ_packed=np.stack(occ),
                        meta=np.array(meta), sha256=np.array(shas),
                        n_cols=m.occupancy.shape[1])


def record(vec, n, steps, seed, keep_every):
    import color_rl.vecenv as vmod
    with reference_rng_proxy(vmod):
        s0 = vec.reset_all(seed)
    rew, ev, dn, tr, obs_steps, st, ss = [], [], [], [], [], [], []
    for t in range(steps):
        a = random_actions(seed, np.arange(n), t)
        b = vec.step_batch(a)
        rew.append(b.rewards)
        ev.append(b.events)
        dn.append(b.dones)
        tr.append(b.truncated)
        if t % keep_every == 0 or t == steps - 1:
            obs_steps.append(t)
            st.append(b.states)
            ss.append(b.store_states)
    snap = vec.snapshot_stats()
    return dict(seed=seed, reset_states=s0, rewards=np.array(rew), events=np.array(ev),
                dones=np.array(dn), truncated=np.array(tr), obs_steps=np.array(obs_steps),
                states=np.array(st), store_states=np.array(ss),
                final_x=vec.sim.x.copy(), final_y=vec.sim.y.copy(),
                final_heading=vec.sim.heading.copy(),
                rng_ctr=np.array([vec.sim._rngs[i].ctr for i in range(n)], dtype=np.uint64),
                episodes=np.array([c.episodes for c in snap.per_copy]),
                arrivals=np.array([c.arrivals for c in snap.per_copy]),
                return_sum=np.array([c.return_sum for c in snap.per_copy]),
                recent_returns=np.array(snap.recent_returns))


def main():
    O.load_lib()
    O.import_reference(5 + R)
    from color_rl.mapgen import generate_maps
    from color_rl.sim.gridmap import GridMap
    from color_rl.sim.params import DiversityRanges, EnvConfig, LidarConfig, SimParams
    from color_rl.vecenv import VecEnv
    from color_rl import kernels
    from color_rl.replay import ReplayBuffer

    texts = [m.to_text() for m in generate_maps(16, seed=0, size_cm=366, density=0.08)]
    save_maps(texts)
    maps = [GridMap.from_text(t) for t in texts]
    cfg = EnvConfig(lidar=LidarConfig(n_beams=R))

    vec = VecEnv(maps[:1], 16, DiversityRanges(), cfg)
    np.savez_compressed(os.path.join(OUT, "traj_cfg1.npz"),
                        **record(vec, 16, 1000, 1234, 50))
    vec = VecEnv(maps, 256, DiversityRanges.around(SimParams(), 0.3), cfg)
    np.savez_compressed(os.path.join(OUT, "traj_cfg2.npz"),
                        **record(vec, 256, 100, 777, 33))

    # kernel goldens on free poses of every map
    rng = np.random.default_rng(2024)
    occ = np.stack([m.occupancy for m in maps]).astype(np.uint8)
    edt = np.stack([m.edt_cells() for m in maps])
    qx, qy, qh, qm = [], [], [], []
    for m in range(16):
        free = np.argwhere(occ[m] == 0)
        for iy, ix in free[rng.integers(0, len(free), 32)]:
            qx.append(ix + rng.random()); qy.append(iy + rng.random())
            qh.append(rng.uniform(-np.pi, np.pi)); qm.append(m)
    qx, qy, qh, qm = (np.array(v) for v in (qx, qy, qh, qm))
    ang = qh[:, None] + cfg.lidar.beam_offsets()[None, :]   # core.py:224
    px, py = np.repeat(qx, R), np.repeat(qy, R)
    dx, dy, mi = np.cos(ang).ravel(), np.sin(ang).ravel(), np.repeat(qm, R)
    cy = kernels.get_backend("cy")
    outs = {f"out_{int(mr)}": kernels.cast_rays(occ, edt, mi, px, py, dx, dy, 1.0, mr, backend=cy)
            for mr in (150.0, 300.0, 500.0)}
    disc = kernels.disc_collides(occ, mi[::R], px[::R], py[::R], np.full(len(px) // R, 9.0), 1.0,
                                 backend=cy)
    np.savez_compressed(os.path.join(OUT, "rays16.npz"), qx=qx, qy=qy, qh=qh, qmap=qm,
                        disc=disc, **outs)

    # replay: ring contents + Philox-stream samples
    buf = ReplayBuffer(capacity=1000, state_dim=4)
    for start in range(0, 1500, 100):
        base = np.arange(start, start + 100, dtype=np.float32)
        buf.append_batch(np.tile(base[:, None], (1, 4)), base.astype(np.int64) % 5, base * 0.5,
                         np.tile(base[:, None], (1, 4)) + 0.25, base.astype(np.int64) % 7 == 0)
    g = PhiloxStream(99, 3, tag=2)
    samples = [buf.sample(256, g) for _ in range(4)]
    np.savez_compressed(os.path.join(OUT, "replay.npz"),
                        states=np.stack([s.states for s in samples]),
                        actions=np.stack([s.actions for s in samples]),
                        rewards=np.stack([s.rewards for s in samples]),
                        dones=np.stack([s.dones for s in samples]), seed=99, stream=3)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
