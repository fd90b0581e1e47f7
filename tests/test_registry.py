"""DeviceRegistry: device residency follows the wrapped
registry's lease / eviction lifecycle (model.py:311-421).  Host logic with a
fake registry and fake uploads on CPU; the real upload path is exercised by
test_gpu_parity.py::test_device_registry_residency."""

import numpy as np
import pytest

from paper_2605_08699_b200.registry import DeviceRegistry, _scene_bytes


class FakePrims:
    def __init__(self, n):
        self.means = np.zeros((n, 3))
        self.sh_coeffs = np.zeros((n, 16, 3))


class FakeScene:
    def __init__(self, prims):
        self.device_bytes = _scene_bytes(prims)


class FakeRegistry:
    """The reference ModelRegistry's interface, in memory."""

    def __init__(self, sizes):
        self.sizes = sizes
        self.loaded, self.refs, self.loads = {}, {}, 0

    def acquire(self, mid):
        if mid not in self.sizes:
            raise KeyError(mid)
        if mid not in self.loaded:
            self.loaded[mid] = FakePrims(self.sizes[mid])
            self.loads += 1
        self.refs[mid] = self.refs.get(mid, 0) + 1
        return self.loaded[mid]

    def release(self, mid):
        self.refs[mid] -= 1

    def evict_inactive(self, now=None):
        gone = [m for m in self.loaded if self.refs.get(m, 0) == 0]
        for m in gone:
            del self.loaded[m]
        return gone

    def snapshot(self):
        return [{"id": m} for m in sorted(self.sizes)]


@pytest.fixture
def reg(monkeypatch):
    r = DeviceRegistry(FakeRegistry({"a": 1000, "b": 2000, "c": 1500}), device=0)
    freed = []
    monkeypatch.setattr(r, "_upload", lambda prims: FakeScene(prims))
    monkeypatch.setattr(r, "_free", lambda prims: freed.append(prims))
    r.freed = freed
    return r


def test_upload_once_per_host_load(reg):
    p1 = reg.acquire("a")
    p2 = reg.acquire("a")
    assert p1 is p2 and reg.uploads == 1
    reg.release("a")
    reg.release("a")
    with reg.lease("a") as p3:
        assert p3 is p1
    assert reg.uploads == 1
    assert reg.device_bytes() == _scene_bytes(p1)
    assert [r["device_resident"] for r in reg.snapshot()] == [True, False, False]


def test_eviction_frees_device_copy(reg):
    with reg.lease("a"):
        pass
    with reg.lease("b"):
        assert reg.evict_inactive() == ["a"]  # b is leased
    assert len(reg.freed) == 1 and reg.device_bytes() > 0
    assert reg.evict_inactive() == ["b"]
    assert reg.device_bytes() == 0
    # host reload after eviction -> fresh upload
    with reg.lease("a"):
        pass
    assert reg.uploads == 3


def test_device_budget_lru_respects_leases(reg):
    reg.max_device_bytes = _scene_bytes(FakePrims(1000)) + _scene_bytes(FakePrims(2000))
    with reg.lease("a"):
        with reg.lease("b"):
            pass
        # c does not fit: b (no lease) is freed first, a is leased and stays
        with reg.lease("c"):
            pass
    assert reg.device_evictions == 1
    rows = {r["id"]: r["device_resident"] for r in reg.snapshot()}
    assert rows == {"a": True, "b": False, "c": True}


def test_failed_upload_releases_lease(reg, monkeypatch):
    def boom(prims):
        raise RuntimeError("upload failed")
    monkeypatch.setattr(reg, "_upload", boom)
    with pytest.raises(RuntimeError):
        reg.acquire("a")
    assert reg.registry.refs["a"] == 0 and reg._leases["a"] == 0
