"""B200-native Sparrow hot path (arXiv 2305.04180, "Color"): the vectorized
environment step with fused auto-reset and the Sharer replay ring, as CUDA
kernels for sm_100a behind a C-ABI (include/sparrow.h, _lib/libsparrow.so).

Drop-in names of the reference package ``color_rl``:
  VecEnv, StepBatch, StatsSnapshot, CopyStats          (color_rl.vecenv)
  ReplayBuffer, TransitionBatch, BufferNotReady        (color_rl.replay)
  GridMap, MapError, DiversityRanges, SimParams,
  LidarConfig, EnvConfig, Event, EpisodeTerminated     (color_rl.sim)
  kernels (BACKEND_NAME = "cuda": cast_rays, disc_collides)  (color_rl.kernels seam)
Submodules beyond the hot path:
  asl       Q-net, DDQN + fused Adam + CUDA-graphed update, VEM, TFM, Sharer, session
  evaluate  greedy evaluation (evaluate_params, EvalReport, summarize_rates)
  mapgen    procedural arenas, host side (generate_map(s), write_maps)
"""

from paper_2305_04180_b200.sim import (  # noqa: F401
    ACTION_TABLE,
    DiversityRanges,
    EnvConfig,
    EpisodeTerminated,
    Event,
    GridMap,
    LidarConfig,
    MapError,
    SimParams,
)
from paper_2305_04180_b200.replay import (  # noqa: F401
    BufferNotReady,
    PhiloxGenerator,
    ReplayBuffer,
    TransitionBatch,
)
from paper_2305_04180_b200.vecenv import CopyStats, StatsSnapshot, StepBatch, VecEnv  # noqa: F401

__version__ = "0.1.0"
