"""ABR-mixed rung sequences for BASELINE config 5 ("an
ABR-mixed sequence precomputed with the reference LatencyAbr and
TokenBucketShaper on a seeded bandwidth trace (virtual time)").

For each of the 64 sessions (session i = pose trace seed i, as bench.py):
  * a seeded bandwidth trace (harness.py BandwidthTrace: a log-space random
    walk of the rate between 2 and 80 Mbit/s, a new rate every 0.5-2 s),
  * the session's movement trace (paper_2605_08699_b200.synth.pose_trace,
    30 Hz) for the panning flag (harness.py:250-254),
  * payload bytes of each response = the rung's starting expected size
    times a seeded log-normal factor (sigma 0.25) -- an open-loop size model
    standing in for the JPEG sizes,
and the reference's own LatencyAbr + TokenBucketShaper are stepped exactly as
harness.run_session does on its virtual clock (harness.py:296-365):
t_send = max(entry_t, completion); t_recv = shaper.deliver(bytes, t_send) +
RTT; abr.on_response(bytes, t_recv - t_send, panning).  The level chosen for
every frame is recorded.  The ladder is config 3's (1080p / 720p / 540p /
360p, ladder_from_config, abr.py:92-100).  The GPU box has no
/root/reference: bench.py and the tests read the committed abr_sequence.json.

    python tests/golden/make_abr_sequence.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent.parent))

import numpy as np  # noqa: E402

from splatstream.abr import LatencyAbr, ladder_from_config  # noqa: E402
from splatstream.harness import (DEFAULT_VIRTUAL_RTT, BandwidthEntry, BandwidthTrace,  # noqa: E402
                                 MovementEntry, TokenBucketShaper, _is_panning)

from paper_2605_08699_b200.synth import ladder_1080p, pose_trace  # noqa: E402

N_SESSIONS = 64
FRAMES = 300
RUNGS = ladder_1080p()


def bandwidth_trace(seed: int, seconds: float) -> BandwidthTrace:
    rng = np.random.default_rng(10_000 + seed)
    t, lr, out = 0.0, np.log(rng.uniform(4.0, 40.0)), []
    while t < seconds:
        out.append(BandwidthEntry(t_ms=round(t * 1000.0, 3),
                                  rate_kbps=round(float(np.exp(lr)) * 1000.0, 3)))
        t += float(rng.uniform(0.5, 2.0))
        lr = float(np.clip(lr + rng.normal(0.0, 0.6), np.log(2.0), np.log(80.0)))
    return BandwidthTrace(entries=tuple(out))


def session_levels(seed: int):
    ladder = ladder_from_config(RUNGS)
    expected = [p.expected_size_bytes for p in ladder.profiles]
    abr = LatencyAbr(ladder)
    trace = pose_trace(FRAMES, seed=seed)
    bw = bandwidth_trace(seed, trace[-1].t_ms / 1000.0 + 60.0)
    shaper = TokenBucketShaper(bw)
    rng = np.random.default_rng(20_000 + seed)
    prev, completion, levels = None, 0.0, []
    for tp in trace:
        entry = MovementEntry(t_ms=tp.t_ms, azimuth_deg=tp.azimuth_deg,
                              elevation_deg=tp.elevation_deg, translation=tuple(tp.translation))
        level = abr.profile().level
        levels.append(level)
        t_send = max(tp.t_ms / 1000.0, completion)
        nbytes = max(1, int(expected[level] * float(np.exp(rng.normal(0.0, 0.25)))))
        t_recv = shaper.deliver(nbytes, t_send) + DEFAULT_VIRTUAL_RTT
        panning = _is_panning(prev, entry)
        prev = entry
        completion = t_recv
        abr.on_response(nbytes, t_recv - t_send, panning)
    return levels, len(bw.entries)


def main():
    sessions = []
    hist = [0] * len(RUNGS)
    for i in range(N_SESSIONS):
        lv, nbw = session_levels(i)
        for x in lv:
            hist[x] += 1
        sessions.append({"index": i, "levels": "".join(str(x) for x in lv),
                         "bandwidth_changes": nbw})
    out = {"what": __doc__.split("\n\n")[0], "rungs": RUNGS, "frames_per_session": FRAMES,
           "level_histogram": hist, "sessions": sessions}
    (HERE / "abr_sequence.json").write_text(json.dumps(out, indent=1))
    print("level histogram", hist)


if __name__ == "__main__":
    main()
