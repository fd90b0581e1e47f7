"""Scene load on the GPU: PLY bytes -> resident scene.

The reference's registry loads a model with
``activate(parse_ply(rec.ply_path.read_bytes()))`` (model.py:354): a numpy
parse of the float32 vertex table (model.py:169-208), finiteness checks and
the activation (model.py:211-252), all on the host, then every render reads
those f64 arrays again.  ``load_ply`` does the same in one pass on the device
(``gsr_scene_create_ply``, csrc/ply.cu): the header is parsed on the host with
the reference's error classes and messages, the vertex table is copied to HBM
and decoded, checked and activated by one kernel straight into the scene the
renderer reads.  Every array equals the reference's bit for bit, including
np.exp / scipy expit / np.log (restated in csrc/libm_restated.cuh).

``load_ply`` returns a ``DeviceActivatedPrimitives``: it has the
``ActivatedPrimitives`` interface (model.py:89-102) -- the host arrays are
read back from the device on first access -- and carries its device scene, so
``render_*`` / ``RenderPipeline`` / ``DeviceRegistry`` use it without an
upload.  ``parse_ply_header`` exposes the host header parse alone.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .synth import PLY_REQUIRED, PLY_REST, ActivatedPrimitives


class ModelError(Exception):
    """model.py:40-41."""


class MalformedHeader(ModelError):
    """model.py:44-45."""


class MissingProperty(ModelError):
    """model.py:48-49."""


class TruncatedBody(ModelError):
    """model.py:52-53."""


class NonFiniteAttribute(ModelError):
    """model.py:56-57."""


@dataclass(frozen=True)
class PlyHeader:
    """What _parse_header + parse_ply's checks establish (model.py:105-186)."""

    count: int
    body_offset: int
    n_props: int
    has_rest: bool
    columns: dict          # loader property -> column index in the vertex table

    @property
    def body_bytes(self) -> int:
        return self.count * self.n_props * 4


def _as_bytes(source) -> bytes:
    if isinstance(source, (str, Path)):
        return Path(source).read_bytes()
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source) if not isinstance(source, bytes) else source
    raise TypeError("source must be PLY bytes or a path")


def parse_ply_header(source) -> PlyHeader:
    """Header + property + length checks of parse_ply, on the host (no device).

    Raises MalformedHeader / MissingProperty / TruncatedBody with the
    reference's messages.
    """
    data = _as_bytes(source)
    info = _lib.GsrPlyInfo()
    lib = _lib.load()
    _lib.check(lib.gsr_ply_parse_header(data, len(data), ctypes.byref(info)))
    names = PLY_REQUIRED + PLY_REST
    return PlyHeader(count=int(info.count), body_offset=int(info.body_offset),
                     n_props=int(info.n_props), has_rest=bool(info.has_rest),
                     columns={n: int(info.col[i]) for i, n in enumerate(names)
                              if info.col[i] >= 0})


_ATTRS = {"means": (0, (3,)), "scales": (1, (3,)), "rotations": (2, (4,)),
          "opacities": (3, ()), "colors_dc": (4, (3,)), "sh_coeffs": (5, (16, 3))}


class DeviceActivatedPrimitives:
    """ActivatedPrimitives (model.py:89-102) resident in HBM.

    Attribute arrays are read back (f64, the reference's shapes) on first
    access and cached; ``scene`` is the render path's device copy.
    """

    def __init__(self, scene, load_stats: dict | None = None):
        self.scene = scene                 # render.DeviceScene
        self.device = scene.device
        self.load_stats = load_stats or {}
        self._host: dict = {}
        self._lock = threading.Lock()

    @property
    def count(self) -> int:
        return int(self.scene.count)

    def _read(self, name: str) -> np.ndarray:
        with self._lock:
            arr = self._host.get(name)
            if arr is None:
                if self.scene.closed:
                    raise _lib.RenderError("device scene was freed before its arrays were read")
                which, tail = _ATTRS[name]
                arr = np.empty((self.count,) + tail, dtype=np.float64)
                lib = _lib.load()
                _lib.check(lib.gsr_scene_read(self.scene.handle, which, _lib.ptr(arr)),
                           "gsr_scene_read")
                arr.setflags(write=False)  # primitives are immutable (model.py:92)
                self._host[name] = arr
            return arr

    means = property(lambda self: self._read("means"))
    scales = property(lambda self: self._read("scales"))
    rotations = property(lambda self: self._read("rotations"))
    opacities = property(lambda self: self._read("opacities"))
    colors_dc = property(lambda self: self._read("colors_dc"))
    sh_coeffs = property(lambda self: self._read("sh_coeffs"))

    def materialize(self) -> ActivatedPrimitives:
        """Host copy as the reference's ActivatedPrimitives."""
        return ActivatedPrimitives(**{n: np.array(self._read(n)) for n in _ATTRS})

    def release_device(self) -> None:
        """Free the device scene, keeping the object usable (arrays read first)."""
        for n in _ATTRS:
            self._read(n)
        self.scene.close()


def load_ply(source, device: int | None = None, stats: dict | None = None
             ) -> DeviceActivatedPrimitives:
    """activate(parse_ply(data)) on the device (model.py:169-252, 354).

    `source`: PLY bytes or a path.  Raises the reference's MalformedHeader /
    MissingProperty / TruncatedBody / NonFiniteAttribute; RenderError when no
    device is available (there is no CPU fallback).  If `stats` is a dict it
    receives the load timings (h2d_ms, kernel_ms, total_ms, bytes).
    """
    from .render import DeviceScene, _default_device
    data = _as_bytes(source)
    dev = _default_device if device is None else int(device)
    lib = _lib.load()
    h = ctypes.c_void_p()
    st = _lib.GsrPlyStats()
    _lib.check(lib.gsr_scene_create_ply(ctypes.byref(h), dev, data, len(data), ctypes.byref(st)),
               "gsr_scene_create_ply")
    scene = DeviceScene.from_handle(h, dev)
    d = st.as_dict()
    if stats is not None:
        stats.update(d)
    return DeviceActivatedPrimitives(scene, d)


__all__ = ["ModelError", "MalformedHeader", "MissingProperty", "TruncatedBody",
           "NonFiniteAttribute", "PlyHeader", "parse_ply_header", "DeviceActivatedPrimitives",
           "load_ply"]
