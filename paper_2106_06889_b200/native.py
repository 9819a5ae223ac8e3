"""Native TSV rendering and SHA-256 output digests (render.cpp via the C-ABI).

`NativeDict(blob).render(compact)` is byte-identical to the reference's
`render(run_task(...), dictionary)` (`tasks.py:233-263`) and
`NativeDict(blob).digest(compact)` is the sha256 of that text — the CLI
manifest's `outputDigest` (`cli.py:121-133`) — without building Python
containers or the text.  Host-only code: works without a GPU, and on any
render-ordered `Compact` (device results, oracle results, combined shards).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._abi import TASK_IDS, Compact, GtView, raise_for_status
from .device import lib


def _ptr(a: np.ndarray | None, dtype, keep: list):
    if a is None:
        return None
    b = np.ascontiguousarray(a, dtype=dtype)
    keep.append(b)
    ctype = C.c_uint64 if dtype == np.uint64 else C.c_uint32
    return b.ctypes.data_as(C.POINTER(ctype))


def view_of(c: Compact):
    """A gt_view over a Compact's arrays (typed copies kept alive in the
    returned list)."""
    keep: list = []
    v = GtView()
    v.task = TASK_IDS[c.task]
    v.seq_len = c.seq_len
    v.wbits = c.wbits
    v.n_groups = c.n_groups
    v.n = c.n
    v.group_off = _ptr(c.group_off, np.uint64, keep)
    v.group_id = _ptr(c.group_id, np.uint32, keep)
    v.group_key = _ptr(c.group_key, np.uint64, keep)
    v.group_gram = _ptr(c.group_gram, np.uint32, keep)
    v.id = _ptr(c.id, np.uint32, keep)
    v.key = _ptr(c.key, np.uint64, keep)
    v.gram = _ptr(c.gram, np.uint32, keep)
    v.count = _ptr(c.count, np.uint64, keep)
    return v, keep


class NativeDict:
    """Word strings of a GTDC blob for native rendering (gt_dict)."""

    def __init__(self, blob: bytes):
        self._h = None
        h = C.c_void_p()
        st = lib().gt_dict_open(bytes(blob), len(blob), C.byref(h))
        raise_for_status(st, "not a GTDC blob")
        self._h = h

    def render(self, c: Compact) -> str:
        v, keep = view_of(c)
        p, n = C.c_void_p(), C.c_uint64()
        raise_for_status(lib().gt_render_view(self._h, C.byref(v), C.byref(p), C.byref(n)), "render failed")
        try:
            # (ctypes.string_at takes a C int size: > 2 GiB outputs need a view)
            return bytes((C.c_char * n.value).from_address(p.value)).decode("utf-8") if n.value else ""
        finally:
            lib().gt_free_text(p)

    def digest(self, c: Compact) -> tuple[str, int]:
        """(sha256 hex of the rendering, its byte length)."""
        v, keep = view_of(c)
        out, n = C.create_string_buffer(32), C.c_uint64()
        raise_for_status(lib().gt_digest_view(self._h, C.byref(v), out, C.byref(n)), "digest failed")
        return out.raw.hex(), n.value

    def close(self) -> None:
        if self._h is not None:
            lib().gt_dict_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sha256(data: bytes) -> str:
    out = C.create_string_buffer(32)
    lib().gt_sha256(data, len(data), out)
    return out.raw.hex()
