"""Greedy-policy evaluation on the GPU.

Drop-in for the reference's ``color_rl.evaluate``
(``pkg/src/color_rl/evaluate.py:22-133``). Each map gets ``episodes_per_map``
parallel copies, and every copy runs exactly one scored episode. Parameters
stay at their nominal values unless a randomization fraction is requested.
Timeouts count as failures. The first-episode latch is kept by the step
kernel (``first_event/first_return/first_steps``, ``vecenv.py:134-141``).

The per-step loop runs on the device: the fused actor kernel (Q-net forward
+ argmax, ties to the lowest index as ``np.argmax``) and the fused env step,
``check_every`` steps per CUDA graph replay. No host round trip happens
except the done-check, which reads one count of still-running first episodes
every ``check_every`` steps. Outcomes are latched, so stepping past the
moment every copy has finished cannot change the report. The loop therefore
gives the same report as the reference's check-every-step loop
(``evaluate.py:99-105``).

``fused=True`` puts every map in ONE VecEnv (one launch per step for the
whole map set) instead of one VecEnv per map. Its per-copy random streams
differ from the per-map layout, because the reference seeds each map's env
separately. Use it for arrival rates at scale. The default per-map layout
is the reference's, stream for stream.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .sim import DiversityRanges, EnvConfig, Event, SimParams
from .vecenv import VecEnv

__all__ = ["MapEval", "EvalReport", "evaluate_params", "summarize_rates"]


@dataclass
class MapEval:  # evaluate.py:22-42
    """Outcome counts of one map's scored first episodes."""
    name: str
    episodes: int
    arrivals: int
    collisions: int
    timeouts: int
    mean_return: float
    mean_steps: float

    @property
    def arrival_rate(self) -> float:
        return self.arrivals / self.episodes

    _KEYS = ("name", "episodes", "arrivals", "collisions", "timeouts", "arrival_rate",
             "mean_return", "mean_steps")

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in self._KEYS}


# render() columns: (header, width, row formatter) -- evaluate.py:72-85
_COLUMNS = (("map", -28, lambda r: r.name), ("episodes", 8, lambda r: f"{r.episodes}"),
            ("arrived", 8, lambda r: f"{r.arrivals}"), ("rate", 6, lambda r: f"{r.arrival_rate:.2f}"),
            ("return", 9, lambda r: f"{r.mean_return:.2f}"), ("steps", 7, lambda r: f"{r.mean_steps:.1f}"))


def _cells(values) -> str:
    out = []
    for (_, w, _f), v in zip(_COLUMNS, values):
        out.append(v.ljust(-w) if w < 0 else v.rjust(w))
    return " ".join(out)


@dataclass
class EvalReport:  # evaluate.py:45-85
    """Per-map results of one evaluation seed, pooled on demand."""
    seed: int
    results: list = field(default_factory=list)

    @property
    def episodes(self) -> int:
        return sum(r.episodes for r in self.results)

    @property
    def arrival_rate(self) -> float:
        n = self.episodes
        return sum(r.arrivals for r in self.results) / n if n else 0.0

    @property
    def mean_return(self) -> float:
        n = self.episodes
        return sum(r.mean_return * r.episodes for r in self.results) / n if n else 0.0

    def to_dict(self) -> dict:
        return dict(seed=self.seed, arrival_rate=self.arrival_rate,
                    mean_return=self.mean_return, episodes=self.episodes,
                    maps=[r.to_dict() for r in self.results])

    def render(self) -> str:
        lines = [_cells([c[0] for c in _COLUMNS])]
        lines += [_cells([f(r) for _, _, f in _COLUMNS]) for r in self.results]
        pooled = ["pooled", f"{self.episodes}", f"{sum(r.arrivals for r in self.results)}",
                  f"{self.arrival_rate:.2f}", f"{self.mean_return:.2f}"]
        lines.append(_cells(pooled))
        return "\n".join(lines)


def _as_qnet(params, device):
    from .asl import QNet
    if isinstance(params, QNet):
        return params
    # the reference's MlpParams (numpy weights/biases), net.py:29-45
    return QNet.from_numpy(params.weights, params.biases, getattr(params, "version", 0),
                           device=device)


def _map_seed(seed: int, mi: int) -> int:
    return int(np.random.SeedSequence((seed, mi)).generate_state(1)[0])  # evaluate.py:98


def _rollout(env: VecEnv, net, seed: int, horizon: int, check_every: int, graph: bool = True):
    """Greedy first-episode rollout of every copy (evaluate.py:98-106).
    Returns the per-copy (first_event, first_return, first_steps) arrays.

    With ``graph`` (default) a step is the fused actor kernel with exploration
    off (sp_actor_select: forward + argmax, ties to the lowest index) and the
    fused env step, and ``check_every`` (rounded up to even) such steps are
    one CUDA graph replay, outputs alternating between two buffer sets inside
    it.  Between replays the host reads one count (copies still in their first
    episode).  Outcomes are latched, so the steps past the last finish change
    nothing.  ``graph=False``: cuBLAS forward + torch argmax, one step at a
    time."""
    import torch
    states = env.reset_all(seed)
    if not graph:
        for k in range(horizon):
            with torch.no_grad():
                actions = torch.argmax(net.forward(states), dim=1)
            states = env.step_batch(actions).states
            if (k + 1) % check_every == 0 and env.all_first_episodes_done:
                break
    else:
        from .asl import VemSchedule, no_gc, select_actions_fused
        from .replay import PhiloxGenerator
        n = env.n_copies
        greedy = VemSchedule(n, or_init=1, or_final=1, e_min=0.0, e_max=0.0)
        rng = PhiloxGenerator(0, 0)  # draws made but never used: eps = 0
        outs = [env.new_batch(), env.new_batch()]
        acts = torch.empty(n, dtype=torch.int64, device=env.device)
        outs[1].states.copy_(states)
        k_graph = check_every + (check_every & 1)
        select_actions_fused(net, outs[1].states, greedy, 0, rng, out=acts)  # warm the kernel
        side = torch.cuda.Stream(env.device)
        side.wait_stream(torch.cuda.current_stream(env.device))
        g = torch.cuda.CUDAGraph()
        with no_gc(), torch.cuda.graph(g, stream=side):  # no cudaFree by a collection mid-capture
            for i in range(k_graph):
                select_actions_fused(net, outs[(i + 1) & 1].states, greedy, 0, rng, out=acts)
                env.step_device(acts.data_ptr(), outs[i & 1])
        done = 0
        while done < horizon:
            g.replay()
            done += k_graph
            if env.first_pending() == 0:
                break
        torch.cuda.current_stream(env.device).wait_stream(side)
    st = env._per_copy_arrays()
    if (st["first_event"] < 0).any():
        raise RuntimeError("evaluation episodes did not finish within the timeout")
    return st["first_event"], st["first_return"], st["first_steps"]


def _map_eval(name, events, returns, steps) -> MapEval:
    return MapEval(
        name=name,
        episodes=int(len(events)),
        arrivals=int((events == int(Event.ARRIVAL)).sum()),
        collisions=int((events == int(Event.COLLISION)).sum()),
        timeouts=int((events == int(Event.TIMEOUT)).sum()),
        mean_return=float(np.mean(returns)),
        mean_steps=float(np.mean(steps)),
    )


def evaluate_params(params, maps, names, episodes_per_map: int, seed: int,
                    config: EnvConfig | None = None, nominal: SimParams | None = None,
                    randomize_fraction: float = 0.0, kernel_backend=None, *,
                    device=None, fused: bool = False, check_every: int = 8,
                    graph: bool = True) -> EvalReport:
    """evaluate.py:88-123. ``params`` is a QNet, or anything with the
    reference's ``weights``/``biases`` lists (MlpParams)."""
    config = config or EnvConfig()
    nominal = nominal or SimParams()
    ranges = DiversityRanges.around(nominal, randomize_fraction)
    net = _as_qnet(params, device)
    report = EvalReport(seed=seed)
    horizon = config.timeout_steps + 1
    check_every = max(1, int(check_every))
    maps, names = list(maps), list(names)
    if fused and maps:
        n = len(maps) * episodes_per_map
        midx = np.repeat(np.arange(len(maps)), episodes_per_map)
        env = VecEnv(maps, n, ranges, config, map_index=midx, kernel_backend=kernel_backend,
                     device=device, check_actions=False)
        ev, rt, sp = _rollout(env, net, _map_seed(seed, 0), horizon, check_every, graph)
        for mi, name in enumerate(names):
            sl = slice(mi * episodes_per_map, (mi + 1) * episodes_per_map)
            report.results.append(_map_eval(name, ev[sl], rt[sl], sp[sl]))
        return report
    for mi, (grid_map, name) in enumerate(zip(maps, names)):
        env = VecEnv([grid_map], episodes_per_map, ranges, config,
                     kernel_backend=kernel_backend, device=device, check_actions=False)
        ev, rt, sp = _rollout(env, net, _map_seed(seed, mi), horizon, check_every, graph)
        report.results.append(_map_eval(name, ev, rt, sp))
    return report


def summarize_rates(reports) -> dict:
    """Mean/std of pooled arrival rates across seeds (evaluate.py:126-133)."""
    rates = [r.arrival_rate for r in reports]
    return {
        "per_seed": rates,
        "mean": float(np.mean(rates)) if rates else 0.0,
        "std": float(np.std(rates)) if rates else 0.0,
    }
