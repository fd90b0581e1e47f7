"""Session sharding for multi-GPU serving (BASELINE config 5).

Client sessions are independent (server.py:1-7; statelessness test
test_acceptance.py:358-391), so a box with G GPUs serves session i on GPU
i mod G with no data-path collective.  Each GPU keeps replicas of the scenes
its own sessions use (a 6M-Gaussian SH3 scene is 1.8 GB of HBM; config 5's
14 sizes sum to about 8 GB).  This module is host logic only: which sessions
and scenes a rank owns.
"""

from __future__ import annotations

from dataclasses import dataclass

N_SIZES = 14


def config5_scene_size(k: int) -> int:
    """Scene size k of config 5: round(250k * 24^(k/13)), 250k ... 6M."""
    return int(round(250_000 * 24.0 ** (k / 13.0)))


@dataclass(frozen=True)
class Session:
    index: int       # global session id (also the pose-trace seed)
    scene: int       # scene-size index k (config 5: i mod 14)
    gaussians: int


def config5_sessions(n_sessions: int = 64) -> list[Session]:
    return [Session(i, i % N_SIZES, config5_scene_size(i % N_SIZES)) for i in range(n_sessions)]


def shard(items, rank: int, world: int):
    """Round-robin partition: element i belongs to rank i mod world."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} for world size {world}")
    return [x for i, x in enumerate(items) if i % world == rank]


def scenes_for(sessions) -> list[int]:
    """Distinct scene indices a rank must hold, in first-use order."""
    seen, out = set(), []
    for s in sessions:
        if s.scene not in seen:
            seen.add(s.scene)
            out.append(s.scene)
    return out
