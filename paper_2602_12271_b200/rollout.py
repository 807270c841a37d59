"""Real-activation I/O and the autoregressive rollout driver.

* QKV1 problem files -- the reference's flat container (qkv_io.py:1-63): magic
  ``b"QKV1"``, little-endian ``uint32`` header ``(f, h, w, d)``, then Q, K, V as
  row-major float64 ``(f*h*w, d)`` blocks.  ``save_problem`` / ``load_problem``
  write and parse the same bytes and raise ``TensorFileError`` on the same
  conditions (bad magic, truncated header, non-positive header fields, body size
  mismatch); ``load_qkv`` puts a file's Q/K/V on the device as ``(1, 1, N, d)``
  tensors for the operator.
* ``FrameKVCache`` + ``Rollout`` -- the Self-Forcing generation loop the paper
  times (chunks of frames decoded one after another, every chunk's
  queries attending to all frames generated so far).  Each step appends the
  chunk's K/V to a preallocated device cache (one copy kernel, no reallocation)
  and runs the chunked-KV operator on views of the cache: query tiles are the
  last ``q_frames`` tile-rows of the ``f_kv``-frame key grid (layout.py
  ``lower_chunked``), so no padding and no gather.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .layout import VideoShape, aligned_config, make_tile_plan
from .ops import monarch_attention
from .solver import AttentionProblem

QKV_MAGIC = b"QKV1"
_HEAD = struct.Struct("<4I")   # f, h, w, d


class TensorFileError(ValueError):
    """Malformed QKV1 container (qkv_io.py:21-22)."""


def save_problem(problem: AttentionProblem, path) -> None:
    """Write ``problem`` as a QKV1 container (qkv_io.py:25-35)."""
    s = problem.shape
    with open(path, "wb") as fh:
        fh.write(QKV_MAGIC)
        fh.write(_HEAD.pack(s.f, s.h, s.w, problem.head_dim))
        for m in (problem.q, problem.k, problem.v):
            fh.write(np.ascontiguousarray(m, dtype="<f8").tobytes())


def _parse(path) -> tuple[tuple[int, int, int, int], np.ndarray]:
    """Header and the (3, N, d) float64 body of a QKV1 file, validated like qkv_io.py:38-63."""
    raw = np.fromfile(path, dtype=np.uint8)
    if raw[:4].tobytes() != QKV_MAGIC:
        raise TensorFileError(f"bad magic {raw[:4].tobytes()!r} at byte 0, expected {QKV_MAGIC!r}")
    if raw.size < 4 + _HEAD.size:
        raise TensorFileError(f"truncated header: have {raw.size} bytes, need {4 + _HEAD.size}")
    f, h, w, d = _HEAD.unpack_from(raw[4:4 + _HEAD.size].tobytes())
    if min(f, h, w, d) < 1:
        raise TensorFileError(f"invalid header (f,h,w,d) = {(f, h, w, d)} at byte 4")
    n = f * h * w
    need = 4 + _HEAD.size + 3 * n * d * 8
    if raw.size != need:
        short = need - raw.size
        if short > 0:
            raise TensorFileError(f"container holds {raw.size} bytes but header (f,h,w,d)={(f, h, w, d)} "
                                  f"requires {need} ({short} missing)")
        raise TensorFileError(f"container holds {raw.size} bytes but header requires {need} ({-short} trailing)")
    body = raw[4 + _HEAD.size:].view("<f8").reshape(3, n, d)
    return (f, h, w, d), body


def load_problem(path, scale: float | None = None) -> AttentionProblem:
    """Read a QKV1 container into an ``AttentionProblem`` (qkv_io.py:38-63)."""
    (f, h, w, _), body = _parse(path)
    return AttentionProblem(body[0].copy(), body[1].copy(), body[2].copy(), VideoShape(f, h, w), scale=scale)


def load_qkv(path, device, dtype=torch.bfloat16):
    """(q, k, v, shape): a QKV1 file's activations as (1, 1, N, d) device tensors."""
    (f, h, w, _), body = _parse(path)
    t = torch.from_numpy(np.ascontiguousarray(body)).to(device=device, dtype=dtype)
    return t[0][None, None], t[1][None, None], t[2][None, None], VideoShape(f, h, w)


class FrameKVCache:
    """Preallocated (B, H, max_frames*h*w, d) key / value buffers filled frame by frame."""

    def __init__(self, batch: int, heads: int, max_frames: int, h: int, w: int, d: int, dv: int | None = None,
                 device="cuda", dtype=torch.bfloat16):
        self.hw = h * w
        self.max_frames = max_frames
        self.k = torch.empty(batch, heads, max_frames * self.hw, d, device=device, dtype=dtype)
        self.v = torch.empty(batch, heads, max_frames * self.hw, dv or d, device=device, dtype=dtype)
        self.frames = 0

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor) -> None:
        nf = k_new.shape[2] // self.hw
        if k_new.shape[2] != nf * self.hw or v_new.shape[2] != k_new.shape[2]:
            raise ValueError(f"chunk of {k_new.shape[2]} tokens is not a whole number of {self.hw}-token frames")
        if self.frames + nf > self.max_frames:
            raise ValueError(f"cache holds {self.max_frames} frames; {self.frames} + {nf} requested")
        lo, hi = self.frames * self.hw, (self.frames + nf) * self.hw
        self.k[:, :, lo:hi].copy_(k_new)
        self.v[:, :, lo:hi].copy_(v_new)
        self.frames += nf

    def view(self) -> tuple[torch.Tensor, torch.Tensor]:
        n = self.frames * self.hw
        return self.k[:, :, :n], self.v[:, :, :n]

    def reset(self) -> None:
        self.frames = 0


class Rollout:
    """Block-causal chunked decoding: ``step(q, k, v)`` appends the chunk's K/V to the
    cache and returns the chunk's attention output over every cached frame.

    ``tile`` is the plan's neighborhood ``(n_f, n_h, n_w)`` on the (f, h) x (w)
    aligned config -- ``(1, h, w)`` is the paper's (h, w) plan, ``(3, h, w)`` its
    (3h, w) plan; ``n_f`` must divide the chunk length."""

    def __init__(self, h: int, w: int, cache: FrameKVCache, tile=None, iterations: int = 1,
                 scale: float | None = None):
        self.h, self.w = h, w
        self.cache = cache
        self.tile = tuple(tile) if tile is not None else (1, h, w)
        self.iterations = iterations
        self.scale = scale
        self._plans = {}

    def plan(self, kv_frames: int):
        p = self._plans.get(kv_frames)
        if p is None:
            shape = VideoShape(kv_frames, self.h, self.w)
            p = make_tile_plan(shape, aligned_config(shape, ("f", "h")), self.tile)
            self._plans[kv_frames] = p
        return p

    def step(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        self.cache.append(k, v)
        kc, vc = self.cache.view()
        f_kv = self.cache.frames
        return monarch_attention(q, kc, vc, self.plan(f_kv), iterations=self.iterations, scale=self.scale,
                                 kv_frames=f_kv)


def rollout_chunks(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, h: int, w: int, chunk_frames: int,
                   tile=None, iterations: int = 1) -> torch.Tensor:
    """Run a whole (B, H, F*h*w, d) sequence chunk by chunk through a fresh cache and
    return the concatenated block-causal output (each chunk attends to frames <= its own)."""
    hw = h * w
    frames = q.shape[2] // hw
    if frames % chunk_frames:
        raise ValueError(f"{frames} frames do not split into chunks of {chunk_frames}")
    cache = FrameKVCache(q.shape[0], q.shape[1], frames, h, w, k.shape[3], v.shape[3], q.device, q.dtype)
    ro = Rollout(h, w, cache, tile, iterations)
    outs = []
    for c in range(frames // chunk_frames):
        sl = slice(c * chunk_frames * hw, (c + 1) * chunk_frames * hw)
        outs.append(ro.step(q[:, :, sl], k[:, :, sl], v[:, :, sl]))
    return torch.cat(outs, dim=2)


__all__ = ["QKV_MAGIC", "TensorFileError", "save_problem", "load_problem", "load_qkv", "FrameKVCache", "Rollout",
           "rollout_chunks"]
