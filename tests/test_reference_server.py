"""The drop-in inside the reference's own server and registry.

The unmodified reference package (pip-installed into baseline/_ref, which
ships to the GPU box with the repo) serves POST /render through its own
Starlette app (server.py:96-145), ModelRegistry (model.py:311-421) and
request model; INTEGRATION.md's import swap replaces server.py:36's
`render_framebuffer` / `encode_jpeg` with this package's, optionally with
the registry wrapped in DeviceRegistry and the registry's load line
(model.py:354) replaced by `load_ply`.  The JPEG bytes the patched server
returns must equal the unpatched reference server's for the same requests.
Skipped when baseline/_ref is absent.
"""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not (REF / "splatstream" / "server.py").exists():
        pytest.skip("baseline/_ref (the unmodified reference package) is not installed")
    import os
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsr_test_numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    try:
        from starlette.testclient import TestClient  # noqa: F401
        import splatstream.model as M
        import splatstream.server as S
        import splatstream.synth as Y
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"reference server not importable here: {exc}")
    return S, M, Y


REQUESTS = [
    dict(azimuth=0.0, elevation=0.0, translation=(0.0, 0.0, 0.0), jpeg_quality=90),
    dict(azimuth=12.0, elevation=-5.0, translation=(0.1, 0.05, 0.3), jpeg_quality=65),
    dict(azimuth=-20.0, elevation=8.0, translation=(-0.2, 0.0, 0.5), jpeg_quality=35),
]


def _post_all(app, width=320, height=240):
    from starlette.testclient import TestClient
    out = []
    with TestClient(app) as client:
        for i, r in enumerate(REQUESTS):
            body = dict(model_id="demo", fx=300.0, fy=300.0, cx=width / 2, cy=height / 2,
                        width=width, height=height, frame_id=i, **r)
            body["translation"] = list(body["translation"])
            resp = client.post("/render", json=body)
            assert resp.status_code == 200, resp.text
            assert resp.headers["content-type"] == "image/jpeg"
            out.append(resp.content)
        # the server's own error mapping is unchanged: unknown model -> 404,
        # invalid request -> 422
        bad = dict(model_id="nope", fx=300.0, fy=300.0, cx=160.0, cy=120.0, width=320,
                   height=240, frame_id=9, **REQUESTS[0])
        bad["translation"] = list(bad["translation"])
        assert client.post("/render", json=bad).status_code == 404
        bad["model_id"] = "demo"
        bad["width"] = 10
        assert client.post("/render", json=bad).status_code == 422
    return out


def test_reference_server_with_the_drop_in(ref, tmp_path, monkeypatch):
    S, M, Y = ref
    import paper_2605_08699_b200 as g
    root = tmp_path / "models"
    Y.write_demo_model(root / "demo", count=20000, seed=11)
    cfg = S.ServerConfig(model_root=root, inflight_cap=4)

    # the unmodified reference: numba render + Pillow JPEG
    want = _post_all(S.create_app(M.ModelRegistry.from_directory(root), cfg))

    # server.py:36 import swap
    monkeypatch.setattr(S, "render_framebuffer", g.render_framebuffer)
    monkeypatch.setattr(S, "encode_jpeg", g.encode_jpeg)
    got = _post_all(S.create_app(M.ModelRegistry.from_directory(root), cfg))
    assert got == want  # byte-identical JPEG payloads

    # + the registry wrapped so GPU residency follows its leases
    reg = g.DeviceRegistry(M.ModelRegistry.from_directory(root), device=0)
    got = _post_all(S.create_app(reg, cfg))
    assert got == want
    assert reg.uploads == 1

    # + the registry's load line (model.py:354) on the GPU: load_ply
    monkeypatch.setattr(M, "activate", lambda raw: raw)
    monkeypatch.setattr(M, "parse_ply", lambda data: g.load_ply(data))
    got = _post_all(S.create_app(M.ModelRegistry.from_directory(root), cfg))
    assert got == want
