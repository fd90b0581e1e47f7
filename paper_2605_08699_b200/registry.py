"""Device-resident model registry.

The reference keeps activated primitives in host memory inside its
``ModelRegistry`` (model.py:311-421: lazy load on ``acquire``, reference
counts per lease, ``evict_inactive`` after an idle timeout).  ``DeviceRegistry``
wraps any registry with that interface and keeps the GPU copy of each loaded
model in step with it ("persistent VRAM residency"):

* ``acquire``/``lease`` return the host primitives exactly as the wrapped
  registry does, after making sure their scene is resident on this
  registry's device (uploaded once, ``gsr_scene_create``); renders through
  ``render_framebuffer``/``render_view``/``RenderPipeline`` then reuse it.
* ``evict_inactive`` evicts through the wrapped registry and frees the
  device copies of the models it dropped.
* ``max_device_bytes`` bounds the HBM the scenes of this registry use: when
  an upload would exceed it, device copies of models with no outstanding
  lease are freed least-recently-used first (the host copy stays loaded; the
  next acquire re-uploads it).

One registry per GPU (one server process per GPU, or ``set_device``).
"""

from __future__ import annotations

import threading
import time
from collections import OrderedDict


class DeviceRegistry:
    def __init__(self, registry, device: int = 0, max_device_bytes: int | None = None,
                 clock=time.monotonic):
        self.registry = registry
        self.device = int(device)
        self.max_device_bytes = max_device_bytes
        self._clock = clock
        self._lock = threading.Lock()
        self._resident: OrderedDict = OrderedDict()  # model_id -> (prims, DeviceScene)
        self._leases: dict = {}                     # model_id -> outstanding leases
        self.uploads = 0
        self.device_evictions = 0

    # -- device residency ---------------------------------------------------
    def _upload(self, prims):
        from .render import device_scene
        return device_scene(prims, self.device)

    def _free(self, prims):
        from .render import evict
        evict(prims, self.device)

    def device_bytes(self) -> int:
        with self._lock:
            return sum(sc.device_bytes for _, sc in self._resident.values())

    def _make_room(self, incoming: int) -> None:
        """Free LRU device copies without leases until `incoming` more fits."""
        if self.max_device_bytes is None:
            return
        total = sum(sc.device_bytes for _, sc in self._resident.values())
        for mid in list(self._resident):
            if total + incoming <= self.max_device_bytes:
                break
            if self._leases.get(mid, 0) > 0:
                continue
            prims, sc = self._resident.pop(mid)
            total -= sc.device_bytes
            self._free(prims)
            self.device_evictions += 1

    # -- the wrapped registry's interface ------------------------------------
    def acquire(self, model_id: str):
        prims = self.registry.acquire(model_id)
        try:
            with self._lock:
                self._leases[model_id] = self._leases.get(model_id, 0) + 1
                ent = self._resident.get(model_id)
                if ent is not None and ent[0] is prims:
                    self._resident.move_to_end(model_id)
                    return prims
                if ent is not None:  # reloaded on the host since: drop the stale copy
                    self._free(ent[0])
                    del self._resident[model_id]
                self._make_room(_scene_bytes(prims))
                sc = self._upload(prims)
                self._resident[model_id] = (prims, sc)
                self.uploads += 1
                return prims
        except Exception:
            with self._lock:
                self._leases[model_id] -= 1
            self.registry.release(model_id)
            raise

    def release(self, model_id: str) -> None:
        self.registry.release(model_id)
        with self._lock:
            if self._leases.get(model_id, 0) > 0:
                self._leases[model_id] -= 1

    def lease(self, model_id: str):
        return _Lease(self, model_id)

    def evict_inactive(self, now: float | None = None) -> list:
        evicted = self.registry.evict_inactive(now)
        with self._lock:
            for mid in evicted:
                ent = self._resident.pop(mid, None)
                if ent is not None:
                    self._free(ent[0])
        return evicted

    def snapshot(self) -> list:
        rows = self.registry.snapshot()
        with self._lock:
            for r in rows:
                r["device_resident"] = r.get("id") in self._resident
        return rows


class _Lease:
    def __init__(self, reg: DeviceRegistry, model_id: str):
        self.reg, self.model_id = reg, model_id

    def __enter__(self):
        return self.reg.acquire(self.model_id)

    def __exit__(self, *exc):
        self.reg.release(self.model_id)
        return False


def _scene_bytes(prims) -> int:
    """Device bytes gsr_scene_create will allocate (SoA planes, f32 SH)."""
    own = getattr(prims, "scene", None)  # load_ply: already resident
    if own is not None and hasattr(own, "device_bytes") and not getattr(own, "closed", False):
        return int(own.device_bytes)  # (once evicted, the re-upload's size is estimated below)
    n = int(prims.means.shape[0])
    stride = (max(n, 1) + 31) // 32 * 32
    sh = getattr(prims, "sh_coeffs", None)
    # means/scales/rotations/rsq f64, opacity + dc f32, opacity f64, the (x, y, z, 0)
    # f64 gather copy of the means, f32 SH rows
    return stride * (11 * 8 + 4 + 12 + 8 + 32 + (192 if sh is not None else 0))
