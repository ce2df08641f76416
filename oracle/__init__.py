"""fp64 CPU oracle for the continual-convolution step (arXiv 2204.03418).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2204_03418_b200`` never imports it, and
the C source (``co_oracle.c``) shares no code with the CUDA path.

This module is a thin ctypes wrapper (numpy in, numpy out) around
``co_oracle.c``; every numeric result comes from the C code, whose functions
cite the passages of PAPER.md they follow.  Arrays use the paper's dimension
order (Assumption 1): step ``(B, C, S1, S2)``, clip
``(B, C, T, S1, S2)``, weights ``(Cout, Cin/g, kt, kh, kw)``; absent spatial
axes have size 1 (Conv1d inputs are passed as ``(B, C, S1)`` or ``(B, C)`` and
reshaped here).

"parity unpinned" items: none at function level.  ``head`` (the ring
position of the next output to complete) is pinned by observation in
tests/test_oracle_pins.py (``test_head_is_next_output_index``): from the delay
on it equals the number of Ready outputs emitted so far mod R, and canonical
slot 0 equals PyTorch's partial batch column of that index.

``CO_ORACLE_LIB`` (test infrastructure only, scripts/oracle_mutants.py): load
this prebuilt oracle library instead of building ``liboracle.so`` -- the
mutation check runs the pins against deliberately broken oracles.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "co_oracle.c")
_HDR = os.path.join(_HERE, "co_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile co_oracle.c with gcc (strict IEEE: no fast-math, no FMA contraction)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB) for s in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Desc(C.Structure):
    _fields_ = [("spatial_rank", C.c_int), ("cin", C.c_int), ("cout", C.c_int), ("groups", C.c_int),
                ("kernel", C.c_int * 3), ("stride", C.c_int * 3), ("padding", C.c_int * 3),
                ("dilation", C.c_int * 3), ("in_spatial", C.c_int * 2)]


class _Frame(C.Structure):
    _fields_ = [("p", C.POINTER(C.c_double)), ("sc", C.c_long), ("sh", C.c_long), ("sw", C.c_long)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(os.environ.get("CO_ORACLE_LIB") or build())
            dp = C.POINTER(C.c_double)
            L.or_validate.argtypes = [C.POINTER(_Desc)]
            for fn in ("or_receptive_field", "or_delay", "or_ring_slots"):
                getattr(L, fn).argtypes = [C.POINTER(_Desc)]
            L.or_out_spatial.argtypes = [C.POINTER(_Desc), C.c_int * 2]
            L.or_out_len.argtypes = [C.POINTER(_Desc), C.c_int]
            L.or_column_at.argtypes = [C.POINTER(_Desc), dp, dp, C.POINTER(_Frame), C.c_int, C.c_int, C.c_int]
            L.or_column_at.restype = C.c_double
            L.or_forward.argtypes = [C.POINTER(_Desc), dp, dp, C.c_int, dp, C.c_int, dp]
            L.or_step_new.argtypes = [C.POINTER(_Desc), dp, dp, C.c_int]
            L.or_step_new.restype = C.c_void_p
            L.or_step_free.argtypes = [C.c_void_p]
            L.or_step_clean.argtypes = [C.c_void_p]
            L.or_step_count.argtypes = [C.c_void_p]
            L.or_step_count.restype = C.c_long
            L.or_step_head.argtypes = [C.c_void_p]
            L.or_step_forward.argtypes = [C.c_void_p, dp, C.c_int, dp]
            L.or_step_forward_steps.argtypes = [C.c_void_p, dp, C.c_int, C.c_int, C.c_int,
                                                C.POINTER(C.c_uint8), dp]
            L.or_step_state.argtypes = [C.c_void_p, dp]
            L.or_step_history.argtypes = [C.c_void_p, dp]
            L.or_bruteforce_tick.argtypes = [C.POINTER(_Desc), dp, dp, C.c_int, dp, C.c_int, dp]
            L.or_stack_new.argtypes = [C.c_int, C.POINTER(_Desc), C.POINTER(dp), C.POINTER(dp),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
            L.or_stack_new.restype = C.c_void_p
            L.or_stack_free.argtypes = [C.c_void_p]
            L.or_stack_clean.argtypes = [C.c_void_p]
            L.or_stack_forward.argtypes = [C.c_void_p, dp, C.c_int, dp]
            ip = C.POINTER(C.c_int)
            L.or_accumulate.argtypes = [C.c_int, ip, ip, ip, ip, ip, ip, ip]
            L.or_schedule_ready.argtypes = [C.c_int, C.c_int, C.c_long]
            L.or_bf16_round.argtypes = [C.c_double]
            L.or_bf16_round.restype = C.c_double
            L.or_bf16_round_array.argtypes = [dp, C.c_long]
            L.or_flops_step.argtypes = [C.POINTER(_Desc)]
            L.or_flops_step.restype = C.c_double
            _lib = L
    return _lib


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return C.POINTER(C.c_double)()
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class Desc:
    """Layer descriptor; index 0 of kernel/stride/padding/dilation is temporal."""
    spatial_rank: int
    cin: int
    cout: int
    kernel: Sequence[int]
    stride: Sequence[int] = (1, 1, 1)
    padding: Sequence[int] = (0, 0, 0)
    dilation: Sequence[int] = (1, 1, 1)
    groups: int = 1
    in_spatial: Sequence[int] = (1, 1)

    def c(self) -> _Desc:
        def three(v):
            v = list(v) + [1] * (3 - len(v))
            return (C.c_int * 3)(*v[:3])
        pad = list(self.padding) + [0] * (3 - len(self.padding))
        d = _Desc()
        d.spatial_rank, d.cin, d.cout, d.groups = self.spatial_rank, self.cin, self.cout, self.groups
        d.kernel = three(self.kernel)
        d.stride = three(self.stride)
        d.padding = (C.c_int * 3)(*pad[:3])
        d.dilation = three(self.dilation)
        ins = list(self.in_spatial) + [1] * (2 - len(self.in_spatial))
        d.in_spatial = (C.c_int * 2)(*ins[:2])
        return d

    # derived quantities (all computed by the C oracle)
    @property
    def receptive_field(self) -> int:
        return lib().or_receptive_field(C.byref(self.c()))

    @property
    def delay(self) -> int:
        return lib().or_delay(C.byref(self.c()))

    @property
    def ring_slots(self) -> int:
        return lib().or_ring_slots(C.byref(self.c()))

    @property
    def out_spatial(self):
        out = (C.c_int * 2)()
        lib().or_out_spatial(C.byref(self.c()), out)
        return int(out[0]), int(out[1])

    def out_len(self, T: int) -> int:
        return lib().or_out_len(C.byref(self.c()), T)

    def valid(self) -> bool:
        return lib().or_validate(C.byref(self.c())) == 0

    def flops_step(self) -> float:
        return lib().or_flops_step(C.byref(self.c()))

    @property
    def w_shape(self):
        k = list(self.kernel) + [1] * (3 - len(self.kernel))
        kh = k[1] if self.spatial_rank >= 1 else 1
        kw = k[2] if self.spatial_rank >= 2 else 1
        return (self.cout, self.cin // self.groups, k[0], kh, kw)

    @property
    def in_hw(self):
        s = list(self.in_spatial) + [1, 1]
        return (s[0] if self.spatial_rank >= 1 else 1, s[1] if self.spatial_rank >= 2 else 1)


def _as_step(x: np.ndarray, d: Desc) -> np.ndarray:
    B = x.shape[0]
    H, W = d.in_hw
    return _f64(x).reshape(B, d.cin, H, W)


def _as_clip(x: np.ndarray, d: Desc) -> np.ndarray:
    B, T = x.shape[0], x.shape[2]
    H, W = d.in_hw
    return _f64(x).reshape(B, d.cin, T, H, W)


def _w(W: np.ndarray, d: Desc) -> np.ndarray:
    return _f64(W).reshape(d.w_shape)


def column_at(d: Desc, W, bias, frames, o: int, ho: int, wo: int) -> float:
    """O1 for one output element; frames: list of kt arrays (Cin,S1,S2) or None."""
    Wc, bc = _w(W, d), _f64(bias)
    H, Wd = d.in_hw
    keep, Z = [], (_Frame * len(frames))()
    for k, fr in enumerate(frames):
        if fr is None:
            Z[k].p = C.POINTER(C.c_double)()
            continue
        a = _f64(fr).reshape(d.cin, H, Wd)
        keep.append(a)
        Z[k].p, Z[k].sc, Z[k].sh, Z[k].sw = _dp(a), H * Wd, Wd, 1
    return lib().or_column_at(C.byref(d.c()), _dp(Wc), _dp(bc), Z, o, ho, wo)


def forward(d: Desc, W, bias, x) -> np.ndarray:
    """O2: batch forward of a clip (B,Cin,T,S..) -> (B,Cout,T',S1',S2')."""
    x = _as_clip(x, d)
    B, T = x.shape[0], x.shape[2]
    Tp = d.out_len(T)
    if Tp < 1:
        raise ValueError("insufficient length: T' < 1")
    Ho, Wo = d.out_spatial
    y = np.empty((B, d.cout, Tp, Ho, Wo))
    Wc, bc = _w(W, d), _f64(bias)
    r = lib().or_forward(C.byref(d.c()), _dp(Wc), _dp(bc), B, _dp(x), T, _dp(y))
    assert r == Tp
    return y


class StepMachine:
    """O3/O4/O5: continual step semantics over B streams sharing one clock."""

    def __init__(self, d: Desc, W, bias, B: int):
        self.d, self.B = d, B
        self._W, self._b = _w(W, d), _f64(bias)
        self._h = lib().or_step_new(C.byref(d.c()), _dp(self._W), _dp(self._b), B)
        if not self._h:
            raise ValueError("invalid descriptor")
        self.out_shape = (B, d.cout) + d.out_spatial

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().or_step_free(h)
            self._h = None

    @property
    def n(self) -> int:
        return lib().or_step_count(self._h)

    @property
    def head(self) -> int:
        return lib().or_step_head(self._h)

    def clean_state(self):
        lib().or_step_clean(self._h)

    def forward_step(self, x, update_state: bool = True):
        """Returns the Ready output (B,Cout,S1',S2') or None (Empty)."""
        xp = None if x is None else _as_step(x, self.d)
        y = np.empty(self.out_shape)
        r = lib().or_step_forward(self._h, _dp(xp), int(update_state), _dp(y))
        return y if r else None

    def forward_steps(self, x, pad_end: bool = False, update_state: bool = True):
        """Returns (y compacted (B,Cout,n_ready,S1',S2'), ready_mask)."""
        x = _as_clip(x, self.d)
        T = x.shape[2]
        total = T + (self.d.padding[0] if pad_end else 0)
        mask = np.zeros(total, dtype=np.uint8)
        y = np.zeros((self.B, self.d.cout, max(total, 1)) + self.d.out_spatial)
        n_ready = lib().or_step_forward_steps(self._h, _dp(x), T, int(pad_end), int(update_state),
                                              mask.ctypes.data_as(C.POINTER(C.c_uint8)), _dp(y))
        return np.ascontiguousarray(y[:, :, :n_ready]), mask.astype(bool)

    def history(self) -> np.ndarray:
        """The raw history (f-1, B, Cin, S1, S2): last f-1 padded frames, oldest first."""
        f = self.d.receptive_field
        H, W = self.d.in_hw
        h = np.zeros((max(f - 1, 0), self.B, self.d.cin, H, W))
        if f > 1:
            lib().or_step_history(self._h, _dp(h))
        return h

    def state(self) -> np.ndarray:
        """O5 canonical state (R,B,Cout,S1',S2')."""
        R = self.d.ring_slots
        s = np.zeros((max(R, 0), self.B, self.d.cout) + self.d.out_spatial)
        if R > 0:
            lib().or_step_state(self._h, _dp(s))
        return s


def bruteforce_tick(d: Desc, W, bias, hist) -> Optional[np.ndarray]:
    """O7: sliding-window recomputation; hist (B,Cin,n+1,S..) of all real frames so far."""
    hist = _as_clip(hist, d)
    B, n1 = hist.shape[0], hist.shape[2]
    y = np.empty((B, d.cout) + d.out_spatial)
    Wc, bc = _w(W, d), _f64(bias)
    r = lib().or_bruteforce_tick(C.byref(d.c()), _dp(Wc), _dp(bc), B, _dp(hist), n1, _dp(y))
    return y if r else None


class Stack:
    """O6: sequential stack with Empty short-circuit, ReLU and bf16 activations."""

    def __init__(self, descs: Sequence[Desc], Ws, biases, relu: Sequence[int], round_bf16: Sequence[int], B: int):
        L = len(descs)
        self.descs, self.B = list(descs), B
        self._Ws = [_w(W, d) for W, d in zip(Ws, descs)]
        self._bs = [_f64(b) for b in biases]
        dp = C.POINTER(C.c_double)
        cd = (_Desc * L)(*[d.c() for d in descs])
        wp = (dp * L)(*[_dp(w) for w in self._Ws])
        bp = (dp * L)(*[_dp(b) for b in self._bs])
        self._h = lib().or_stack_new(L, cd, wp, bp, (C.c_int * L)(*relu), (C.c_int * L)(*round_bf16), B)
        if not self._h:
            raise ValueError("invalid stack")
        self.out_shape = (B, descs[-1].cout) + descs[-1].out_spatial

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().or_stack_free(h)
            self._h = None

    def clean_state(self):
        lib().or_stack_clean(self._h)

    def forward_step(self, x, update_state: bool = True):
        xp = _as_step(x, self.descs[0])
        y = np.empty(self.out_shape)
        r = lib().or_stack_forward(self._h, _dp(xp), int(update_state), _dp(y))
        return y if r else None


def accumulate(f: Sequence[int], p: Sequence[int], s: Sequence[int]) -> dict:
    """Principle 5/6 in the worked-example reading (A3)."""
    n = len(f)
    arr = lambda v: (C.c_int * n)(*v)
    s_acc, p_acc, f_acc, d_acc = (C.c_int * n)(), (C.c_int * n)(), (C.c_int * n)(), (C.c_int * n)()
    lib().or_accumulate(n, arr(f), arr(p), arr(s), s_acc, p_acc, f_acc, d_acc)
    out = dict(s_acc=list(s_acc), p_acc=list(p_acc), f_acc=list(f_acc), d_acc=list(d_acc))
    out["s_nn"], out["d_nn"] = out["s_acc"][-1], out["d_acc"][-1]
    return out


def schedule(d_nn: int, s_nn: int, horizon: int):
    return [bool(lib().or_schedule_ready(d_nn, s_nn, t)) for t in range(horizon)]


def bf16_round(a) -> np.ndarray:
    a = _f64(a).copy()
    lib().or_bf16_round_array(_dp(a), a.size)
    return a
