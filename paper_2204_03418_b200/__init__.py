"""B200-native continual-convolution step (Continual Inference Networks, arXiv 2204.03418).

Thin Python binding over the C ABI in ``include/co.h`` (``libco_b200.so``):
argument marshalling only — every step of the path runs in the sm_100a
kernels.  PyTorch supplies device memory and the current CUDA stream.

Method names follow the paper (Principle 2; Principle 3, P:110-120;
Listing 1): ``forward``, ``forward_step``, ``forward_steps``,
``clean_state``, ``delay``, ``receptive_field``.

Tensors keep the paper's logical dimension order (Assumption 1):
a step is ``(B, C, *S)`` and a clip ``(B, C, T, *S)``, stored channels-last in
memory (``torch.channels_last`` for ``(B, C, H, W)``); :func:`channels_last`
converts.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Tuple

import torch

from . import _abi
from ._abi import CoConvDesc, CoInfo, CoMhaDesc, check, lib

__all__ = ["BroadcastReduce", "Conv", "Delay", "Graph", "MultiheadAttention", "Pool", "Residual", "Stack", "channels_last",
           "get_option", "is_channels_last", "load", "options", "set_option"]

_DT = {torch.float32: _abi.CO_F32, torch.bfloat16: _abi.CO_BF16}


def load():
    """Load the native library (raises ImportError if it was not built)."""
    return lib()


def set_option(name: str, value: int) -> None:
    """co_set_option: a documented planner / launch option (include/co.h)."""
    check(lib().co_set_option(name.encode(), int(value)))


def reset_options() -> None:
    """Every option back to its default (co_set_option(NULL, 0))."""
    check(lib().co_set_option(None, 0))


def get_option(name: str) -> int:
    v = C.c_int64()
    check(lib().co_get_option(name.encode(), C.byref(v)))
    return v.value


def all_options() -> dict:
    """Every option's current value (co_option_name enumerates them)."""
    out, i = {}, 0
    while True:
        n = lib().co_option_name(i)
        if not n:
            return out
        out[n.decode()] = get_option(n.decode())
        i += 1


class options:
    """Context manager: ``with co.options(tc_mode=1, pair=2): ...`` sets the
    options and restores the previous values on exit."""

    def __init__(self, **kw):
        self.kw = kw
        self.prev = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.prev[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.prev.items():
            set_option(k, v)
        return False


def channels_last(x: torch.Tensor) -> torch.Tensor:
    """Same logical tensor, channel axis (dim 1) stored innermost."""
    return x.movedim(1, -1).contiguous().movedim(-1, 1)


def is_channels_last(x: torch.Tensor) -> bool:
    return x.movedim(1, -1).is_contiguous()


def _empty_cl(shape: Sequence[int], dtype, device) -> torch.Tensor:
    phys = (shape[0],) + tuple(shape[2:]) + (shape[1],)
    return torch.empty(phys, dtype=dtype, device=device).movedim(-1, 1)


def _device(device) -> torch.device:
    """torch.device with an explicit CUDA index (the current device for "cuda")."""
    d = torch.device(device)
    if d.type == "cuda" and d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def _stream(stream) -> C.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _tup(v, n=3, fill=1):
    if isinstance(v, int):
        return (v,) * n
    v = tuple(v)
    return v + (fill,) * (n - len(v))


def _stream_mask(streams, B: int):
    m = (C.c_uint8 * B)()
    if isinstance(streams, torch.Tensor) and streams.dtype == torch.bool:
        streams = torch.nonzero(streams).flatten().tolist()
    for b in streams:
        if not 0 <= int(b) < B:
            raise ValueError(f"stream {b} out of range")
        m[int(b)] = 1
    return m


def _steps_host(fn, handle, x_host: torch.Tensor, y_host: torch.Tensor, stream):
    """x_host: (T, B, *S, Cin) pinned, time-major; y_host: (>= n_ready, B, *S', Cout) pinned."""
    T = x_host.shape[0]
    mask = (C.c_uint8 * max(T, 1))()
    nr = C.c_int64()
    check(fn(handle, C.c_void_p(x_host.data_ptr()), T, C.c_void_p(y_host.data_ptr()), mask, C.byref(nr),
             _stream(stream)))
    return nr.value, torch.tensor([bool(m) for m in mask[:T]], dtype=torch.bool)


class Conv:
    """A continual convolution layer over ``n_streams`` lockstep streams.

    ``spatial_rank`` 2 is ``co.Conv3d`` (T, S1, S2), 1 is a (T, S1) conv and 0
    is ``co.Conv1d`` over T.  ``weight`` is ``(Cout, Cin/groups, kt, *k_s)`` in
    ``dtype`` (PyTorch's Conv weight layout); ``bias`` is ``(Cout,)``.
    """

    def __init__(self, in_channels: int, out_channels: int, kernel_size, *, weight: Optional[torch.Tensor],
                 bias: Optional[torch.Tensor] = None, stride=1, padding=0, dilation=1, groups: int = 1,
                 spatial_rank: int = 2, in_spatial: Sequence[int] = (1, 1), n_streams: int = 1,
                 dtype: torch.dtype = torch.bfloat16, out_dtype: Optional[torch.dtype] = None,
                 activation: Optional[str] = None, kernel: str = "auto", state_layout: str = "psum",
                 device="cuda", op: str = "conv"):
        self.device = _device(device)
        self.dtype, self.out_dtype = dtype, (out_dtype or dtype)
        self.spatial_rank, self.n_streams = spatial_rank, n_streams
        self.in_channels, self.out_channels = in_channels, out_channels
        d = CoConvDesc()
        d.spatial_rank, d.in_channels, d.out_channels, d.groups = spatial_rank, in_channels, out_channels, groups
        d.kernel = (C.c_int32 * 3)(*_tup(kernel_size))
        d.stride = (C.c_int32 * 3)(*_tup(stride))
        d.padding = (C.c_int32 * 3)(*_tup(padding, fill=0))
        d.dilation = (C.c_int32 * 3)(*_tup(dilation))
        ins = tuple(in_spatial) + (1, 1)
        d.in_spatial = (C.c_int32 * 2)(*ins[:2])
        d.n_streams = n_streams
        d.in_dtype = d.w_dtype = _DT[dtype]
        d.out_dtype = _DT[self.out_dtype]
        d.activation = {None: _abi.CO_ACT_NONE, "none": _abi.CO_ACT_NONE, "relu": _abi.CO_ACT_RELU}[activation]
        d.kernel_choice = _abi.KERNELS[kernel]
        d.state_layout = _abi.STATE_LAYOUTS[state_layout]
        d.op = _abi.OPS[op]
        self.op = op
        self._desc = d
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            if op == "conv":
                w = weight.detach().to(dtype).contiguous()
                on_dev = int(w.is_cuda)
                b = None
                if bias is not None:
                    b = bias.detach().to(torch.float32).to(w.device).contiguous()
                check(lib().co_conv_create(C.byref(d), C.c_void_p(w.data_ptr()),
                                           C.c_void_p(b.data_ptr()) if b is not None else None, on_dev,
                                           C.byref(h)))
            else:
                check(lib().co_conv_create(C.byref(d), None, None, 0, C.byref(h)))
        self._h = h
        info = self.info()
        # the layout the handle keeps ("auto" resolved by the planner; pooling / delay keep frame rings)
        self.state_layout = "raw" if info.state_layout == _abi.CO_STATE_RAW else "psum"
        self.out_spatial: Tuple[int, ...] = tuple(info.out_spatial[:spatial_rank])
        self.in_spatial: Tuple[int, ...] = tuple(ins[:spatial_rank])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().co_conv_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- attributes (Listing 1) ----
    def info(self) -> CoInfo:
        i = CoInfo()
        check(lib().co_conv_info(self._h, C.byref(i)))
        return i

    @property
    def delay(self) -> int:
        return self.info().delay

    @property
    def receptive_field(self) -> int:
        return self.info().receptive_field

    @property
    def kernel_name(self) -> str:
        return lib().co_kernel_name(self._h).decode()

    @property
    def state_layout_used(self) -> str:
        return self.state_layout

    @property
    def kernel_used(self) -> str:
        return _abi.KERNEL_NAMES[self.info().kernel_used]

    def _check_in(self, x: torch.Tensor, clip: bool):
        exp = (self.n_streams, self.in_channels) + ((x.shape[2],) if clip else ()) + self.in_spatial
        if tuple(x.shape) != exp:
            raise ValueError(f"input shape {tuple(x.shape)} != {exp}")
        if x.dtype != self.dtype or not x.is_cuda:
            raise ValueError(f"input must be a CUDA {self.dtype} tensor")
        if not is_channels_last(x):
            raise ValueError("input must be channels-last (use paper_2204_03418_b200.channels_last)")

    # ---- call modes (Principle 2) ----
    def _check_out(self, out: torch.Tensor, shape, dtype):
        """The kernels write `out` through its data pointer: it must be the
        exact (B, C, *S') channels-last tensor of the right dtype and device."""
        if tuple(out.shape) != tuple(shape) or out.dtype != dtype or out.device != self.device:
            raise ValueError(f"out must be a {dtype} {tuple(shape)} tensor on {self.device}, got "
                             f"{out.dtype} {tuple(out.shape)} on {out.device}")
        if not is_channels_last(out):
            raise ValueError("out must be channels-last (use paper_2204_03418_b200.channels_last)")

    def forward_step(self, x: Optional[torch.Tensor], update_state: bool = True, out: Optional[torch.Tensor] = None,
                     stream=None, pad: bool = False) -> Optional[torch.Tensor]:
        """One step.  Returns the emitted output or None (Empty).

        ``x = None`` is an Empty input: it returns None and neither
        computes nor advances the clock, so hand-chained layers
        ``l2.forward_step(l1.forward_step(x))`` short-circuit like a Stack.
        ``pad=True`` (x must be None) feeds one zero padding step instead --
        the end padding of ``pad_end``, which does advance the clock."""
        if x is None and not pad:
            return None
        if x is not None:
            if pad:
                raise ValueError("pad=True takes no input frame")
            self._check_in(x, clip=False)
        shape = (self.n_streams, self.out_channels) + self.out_spatial
        if out is not None:
            self._check_out(out, shape, self.out_dtype)
        y = out if out is not None else _empty_cl(shape, self.out_dtype, self.device)
        r = C.c_int()
        check(lib().co_forward_step(self._h, C.c_void_p(x.data_ptr()) if x is not None else None,
                                    C.c_void_p(y.data_ptr()), int(update_state), C.byref(r), _stream(stream)))
        return y if r.value else None

    def forward_pad_step(self, update_state: bool = True, out: Optional[torch.Tensor] = None, stream=None):
        """One zero padding step (pad_end): ``forward_step(None, pad=True)``."""
        return self.forward_step(None, update_state=update_state, out=out, stream=stream, pad=True)

    def forward_steps(self, x: torch.Tensor, pad_end: bool = False, update_state: bool = True, stream=None):
        """Fold of forward_step over the clip.  Returns (y compacted in
        time, ready_mask) — y is (B, Cout, n_ready, *S')."""
        self._check_in(x, clip=True)
        T = x.shape[2]
        cap = C.c_int64()
        check(lib().co_steps_ready_count(self._h, T, int(pad_end), C.byref(cap)))
        y = _empty_cl((self.n_streams, self.out_channels, cap.value) + self.out_spatial, self.out_dtype, self.device)
        total = T + (self.info().padding_t if pad_end else 0)
        mask = (C.c_uint8 * max(total, 1))()
        nr = C.c_int64()
        check(lib().co_forward_steps(self._h, C.c_void_p(x.data_ptr()), T, C.c_void_p(y.data_ptr()), mask,
                                     C.byref(nr), int(pad_end), int(update_state), _stream(stream)))
        return y, torch.tensor([bool(m) for m in mask[:total]], dtype=torch.bool)

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Batch mode: the regular convolution of the clip; no state."""
        self._check_in(x, clip=True)
        T = x.shape[2]
        Tp = C.c_int64()
        check(lib().co_forward_out_len(self._h, T, C.byref(Tp)))
        if Tp.value < 1:
            raise ValueError(f"clip too short: T'={Tp.value}")
        y = _empty_cl((self.n_streams, self.out_channels, Tp.value) + self.out_spatial, self.out_dtype, self.device)
        check(lib().co_forward(self._h, C.c_void_p(x.data_ptr()), T, C.c_void_p(y.data_ptr()), C.byref(Tp),
                               _stream(stream)))
        return y

    # ---- state (Principle 3) ----
    def clean_state(self, stream=None):
        check(lib().co_state_clean(self._h, _stream(stream)))

    def state_dict_stream(self, stream=None):
        """Canonical state and the clock (co_state_get): PSUM (R, B, *S', Cout)
        fp32; RAW (f-1, B, *S, Cin) in the input dtype (the last f-1 frames);
        pooling (f-1, B, *S', C): the last f-1 spatially reduced frames (MAX in
        the input dtype, -inf padding; AVG fp32 window sums, 0 padding)."""
        nb = C.c_size_t()
        check(lib().co_state_bytes(self._h, C.byref(nb)))
        info = self.info()
        if self.op != "conv":
            st = torch.empty((info.ring_slots, self.n_streams) + self.out_spatial + (self.in_channels,),
                             dtype=self._ring_dtype(), device=self.device)
        elif self.state_layout == "raw":
            st = torch.empty((info.ring_slots, self.n_streams) + self.in_spatial + (self.in_channels,),
                             dtype=self.dtype, device=self.device)
        else:
            st = torch.empty((info.ring_slots, self.n_streams) + self.out_spatial + (self.out_channels,),
                             dtype=torch.float32, device=self.device)
        meta = CoInfo()
        check(lib().co_state_get(self._h, C.c_void_p(st.data_ptr()) if st.numel() else None, nb.value,
                                 C.byref(meta), _stream(stream)))
        return st, meta

    def load_state_stream(self, state: torch.Tensor, meta: CoInfo, stream=None):
        nb = C.c_size_t()
        check(lib().co_state_bytes(self._h, C.byref(nb)))
        if self.op != "conv":
            state = state.to(self._ring_dtype()).contiguous()
        else:
            state = state.to(self.dtype if self.state_layout == "raw" else torch.float32).contiguous()
        check(lib().co_state_set(self._h, C.c_void_p(state.data_ptr()) if state.numel() else None, nb.value,
                                 C.byref(meta), _stream(stream)))

    # ---- per-stream clocks ----
    def clean_streams(self, streams, stream=None):
        """Reset the given streams (indices or a bool mask of length B) to the
        clean state; each restarts its own clock at the next step."""
        m = _stream_mask(streams, self.n_streams)
        check(lib().co_state_clean_streams(self._h, m, _stream(stream)))

    def stream_ready(self) -> torch.Tensor:
        """Per-stream readiness (bool, B) of the last step."""
        m = (C.c_uint8 * self.n_streams)()
        check(lib().co_stream_ready(self._h, m))
        return torch.tensor(list(m), dtype=torch.bool)

    def _ring_dtype(self):
        # pooling ring: spatially reduced frames, MAX in the input dtype, AVG fp32 sums
        return self.dtype if self.op == "max" else torch.float32

    @property
    def n(self) -> int:
        return self.info().n

    @property
    def head(self) -> int:
        return self.info().head

    # ---- host-buffer entry points (e2e) ----
    def forward_steps_host(self, x_host: torch.Tensor, y_host: torch.Tensor, stream=None):
        """Stream T time-major host frames through the layer with overlapped
        copies (co_forward_steps_host).  Returns (n_ready, ready_mask)."""
        return _steps_host(lib().co_forward_steps_host, self._h, x_host, y_host, stream)

    def forward_step_host(self, x_host: torch.Tensor, y_host: torch.Tensor, update_state: bool = True,
                          stream=None) -> bool:
        r = C.c_int()
        check(lib().co_forward_step_host(self._h, C.c_void_p(x_host.data_ptr()), C.c_void_p(y_host.data_ptr()),
                                         int(update_state), C.byref(r), _stream(stream)))
        return bool(r.value)


class Pool(Conv):
    """Continual max / average pooling (``co.MaxPool*`` / ``co.AvgPool*``,
    PAPER.md P:380-394) over ``n_streams`` lockstep streams: a handle of the C
    ABI with ``op`` = MAX / AVG (include/co.h co_op), keeping the RAW frame
    ring.  AVG counts padding as zeros in a divisor of kt kh kw
    (count_include_pad); MAX ignores padding (-inf).  Same call modes, clock and
    state API as :class:`Conv`.
    """

    def __init__(self, kind: str, channels: int, kernel_size, *, stride=1, padding=0, dilation=1,
                 spatial_rank: int = 2, in_spatial: Sequence[int] = (1, 1), n_streams: int = 1,
                 dtype: torch.dtype = torch.bfloat16, out_dtype: Optional[torch.dtype] = None,
                 activation: Optional[str] = None, device="cuda"):
        if kind not in ("max", "avg"):
            raise ValueError("kind must be 'max' or 'avg'")
        super().__init__(channels, channels, kernel_size, weight=None, stride=stride, padding=padding,
                         dilation=dilation, groups=channels, spatial_rank=spatial_rank, in_spatial=in_spatial,
                         n_streams=n_streams, dtype=dtype, out_dtype=out_dtype, activation=activation,
                         kernel="auto", state_layout="raw", device=device, op=kind)
        self.kind = kind


class Delay(Conv):
    """``co.Delay(d)`` over ``n_streams``
    lockstep streams: Empty for the first d steps, then the input of d steps
    ago; batch mode is the identity.  A handle of the C ABI with ``op`` =
    DELAY (a ring of d + 1 frames, copies only)."""

    def __init__(self, delay: int, channels: int, *, spatial_rank: int = 2, in_spatial: Sequence[int] = (1, 1),
                 n_streams: int = 1, dtype: torch.dtype = torch.bfloat16, device="cuda"):
        super().__init__(channels, channels, (delay + 1,) + (1,) * spatial_rank, weight=None,
                         spatial_rank=spatial_rank, in_spatial=in_spatial, n_streams=n_streams, dtype=dtype,
                         out_dtype=dtype, kernel="auto", state_layout="raw", device=device, op="delay")

    def _ring_dtype(self):
        return self.dtype

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Batch mode: the identity on the clip (alignment is structural)."""
        self._check_in(x, clip=True)
        y = _empty_cl(tuple(x.shape), self.dtype, self.device)
        Tp = C.c_int64()
        check(lib().co_forward(self._h, C.c_void_p(x.data_ptr()), x.shape[2], C.c_void_p(y.data_ptr()),
                               C.byref(Tp), _stream(stream)))
        return y


class Residual:
    """``co.Residual(body)`` with Sum (Listing 3; SPEC.md:
    452-458) over the body layers' ``n_streams`` streams: the identity branch
    is delayed to the body's output (``shrink=False``: equal padding, delay =
    the body's; ``shrink=True``: centered, delay (f-1)/2, batch-mode crop), the
    composite is Ready when the body is (Principle 7), and
    ``activation`` ("relu") follows the add.  The body layers are driven by the
    composite: do not step them directly while it is alive."""

    def __init__(self, body: Sequence[Conv], shrink: bool = False, activation: Optional[str] = None):
        self.body = list(body)
        self.shrink = shrink
        arr = (C.c_void_p * len(self.body))(*[c._h.value for c in self.body])
        h = C.c_void_p()
        act = {None: _abi.CO_ACT_NONE, "none": _abi.CO_ACT_NONE, "relu": _abi.CO_ACT_RELU}[activation]
        with torch.cuda.device(self.body[0].device):
            check(lib().co_residual_create(arr, len(self.body), int(shrink), act, C.byref(h)))
        self._h = h
        first, last = self.body[0], self.body[-1]
        self.n_streams, self.channels = first.n_streams, first.in_channels
        self.in_spatial, self.dtype, self.out_dtype, self.device = first.in_spatial, first.dtype, last.out_dtype, first.device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().co_residual_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def delay(self) -> int:
        d, _ = self.delays()
        return d

    def delays(self):
        """(composite delay = the body's, identity-branch delay)."""
        d, k = C.c_int64(), C.c_int64()
        check(lib().co_residual_delay(self._h, C.byref(d), C.byref(k)))
        return d.value, k.value

    def forward_step(self, x: Optional[torch.Tensor], update_state: bool = True, out: Optional[torch.Tensor] = None,
                     stream=None, pad: bool = False) -> Optional[torch.Tensor]:
        """One tick; ``x = None`` is Empty (returns None, no state change),
        ``pad=True`` with ``x = None`` a zero padding step (see Conv.forward_step)."""
        if x is None and not pad:
            return None
        if x is not None:
            self.body[0]._check_in(x, clip=False)
        shape = (self.n_streams, self.channels) + self.in_spatial
        if out is not None:
            self.body[-1]._check_out(out, shape, self.out_dtype)
        y = out if out is not None else _empty_cl(shape, self.out_dtype, self.device)
        r = C.c_int()
        check(lib().co_residual_step(self._h, C.c_void_p(x.data_ptr()) if x is not None else None,
                                     C.c_void_p(y.data_ptr()), int(update_state), C.byref(r), _stream(stream)))
        return y if r.value else None

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Batch mode: body(x) + x (cropped by (f-1)/2 at each end when shrink)."""
        self.body[0]._check_in(x, clip=True)
        T = x.shape[2]
        Tc = T
        for c in self.body:
            t = C.c_int64()
            check(lib().co_forward_out_len(c._h, Tc, C.byref(t)))
            Tc = t.value
        if Tc < 1:
            raise ValueError(f"clip too short: T'={Tc}")
        y = _empty_cl((self.n_streams, self.channels, Tc) + self.in_spatial, self.out_dtype, self.device)
        Tp = C.c_int64()
        check(lib().co_residual_forward(self._h, C.c_void_p(x.data_ptr()), T, C.c_void_p(y.data_ptr()), C.byref(Tp),
                                        _stream(stream)))
        return y

    def clean_state(self, stream=None):
        check(lib().co_residual_clean(self._h, _stream(stream)))


class BroadcastReduce:
    """``co.BroadcastReduce(*branches, reduce=...)`` (PAPER.md P:462-509,
    Listing 3 / Listing 4): the step is broadcast to every
    branch (a :class:`Stack`, or None for the identity), shorter-delay branches
    are delayed to the longest (Principle 7), and the outputs are summed or
    concatenated over channels.  The branch stacks are driven by the composite."""

    def __init__(self, branches: Sequence[Optional["Stack"]], reduce: str = "sum"):
        self.branches = list(branches)
        arr = (C.c_void_p * len(self.branches))(*[(b._h.value if b is not None else None) for b in self.branches])
        h = C.c_void_p()
        check(lib().co_parallel_create(arr, len(self.branches), {"sum": 0, "concat": 1}[reduce], C.byref(h)))
        self._h = h
        first = next(b for b in self.branches if b is not None)
        l0, ll = first.layers[0], first.layers[-1]
        self.n_streams, self.in_channels, self.in_spatial, self.dtype = l0.n_streams, l0.in_channels, l0.in_spatial, l0.dtype
        self.out_spatial, self.out_dtype, self.device = ll.out_spatial, ll.out_dtype, l0.device
        c = C.c_int32()
        check(lib().co_parallel_out_channels(self._h, C.byref(c)))
        self.out_channels = c.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().co_parallel_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def delay(self) -> int:
        d = C.c_int64()
        check(lib().co_parallel_delay(self._h, C.byref(d)))
        return d.value

    def forward_step(self, x: Optional[torch.Tensor], update_state: bool = True, out: Optional[torch.Tensor] = None,
                     stream=None) -> Optional[torch.Tensor]:
        if x is None:                                  # Empty input
            return None
        first = next(b for b in self.branches if b is not None).layers[0]
        first._check_in(x, clip=False)
        shape = (self.n_streams, self.out_channels) + self.out_spatial
        if out is not None:
            first._check_out(out, shape, self.out_dtype)
        y = out if out is not None else _empty_cl(shape, self.out_dtype, self.device)
        r = C.c_int()
        check(lib().co_parallel_step(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), int(update_state),
                                     C.byref(r), _stream(stream)))
        return y if r.value else None

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        T = x.shape[2]
        T_min = T
        for b in self.branches:
            if b is None:
                continue
            t = T
            for c in b.layers:
                v = C.c_int64()
                check(lib().co_forward_out_len(c._h, t, C.byref(v)))
                t = v.value
            T_min = min(T_min, t)
        y = _empty_cl((self.n_streams, self.out_channels, T_min) + self.out_spatial, self.out_dtype, self.device)
        To = C.c_int64()
        check(lib().co_parallel_forward(self._h, C.c_void_p(x.data_ptr()), T, C.c_void_p(y.data_ptr()), C.byref(To),
                                        _stream(stream)))
        return y

    def clean_state(self, stream=None):
        check(lib().co_parallel_clean(self._h, _stream(stream)))


class MultiheadAttention:
    """``co.MultiheadAttention`` in "single-output" mode (
    SPEC.md:357-403) over ``n_streams`` lockstep streams: a step takes x (B, E)
    and, once ``window`` steps are buffered (delay window-1), returns the
    attention of the newest query against the window's keys / values, projected
    by W_o.  Weights in nn.MultiheadAttention's layout (``in_proj_weight``
    (3E, E), ``in_proj_bias``, ``out_proj.weight``, ``out_proj.bias``)."""

    def __init__(self, embed_dim: int, num_heads: int, window: int, *, in_proj_weight: torch.Tensor,
                 out_proj_weight: torch.Tensor, in_proj_bias: Optional[torch.Tensor] = None,
                 out_proj_bias: Optional[torch.Tensor] = None, n_streams: int = 1,
                 out_dtype: torch.dtype = torch.bfloat16, device="cuda"):
        self.E, self.heads, self.window, self.n_streams = embed_dim, num_heads, window, n_streams
        self.out_dtype, self.device = out_dtype, _device(device)
        d = CoMhaDesc()
        d.embed_dim, d.num_heads, d.window, d.n_streams = embed_dim, num_heads, window, n_streams
        d.out_dtype = _DT[out_dtype]
        wq = in_proj_weight.detach().to(torch.bfloat16).contiguous().to(self.device)
        wo = out_proj_weight.detach().to(torch.bfloat16).contiguous().to(self.device)
        bq = None if in_proj_bias is None else in_proj_bias.detach().float().contiguous().to(self.device)
        bo = None if out_proj_bias is None else out_proj_bias.detach().float().contiguous().to(self.device)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(lib().co_mha_create(C.byref(d), C.c_void_p(wq.data_ptr()),
                                      C.c_void_p(bq.data_ptr()) if bq is not None else None, C.c_void_p(wo.data_ptr()),
                                      C.c_void_p(bo.data_ptr()) if bo is not None else None, 1, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().co_mha_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def delay(self) -> int:
        d = C.c_int64()
        check(lib().co_mha_delay(self._h, C.byref(d)))
        return d.value

    def forward_step(self, x: torch.Tensor, update_state: bool = True, out: Optional[torch.Tensor] = None,
                     stream=None) -> Optional[torch.Tensor]:
        """x (B, E) bf16 -> (B, E) or None (Empty)."""
        if x is None:                                  # Empty input
            return None
        if tuple(x.shape) != (self.n_streams, self.E) or x.dtype != torch.bfloat16 or not x.is_contiguous() \
                or x.device != self.device:
            raise ValueError(f"x must be a contiguous bf16 ({self.n_streams}, {self.E}) tensor on {self.device}")
        if out is not None and (tuple(out.shape) != (self.n_streams, self.E) or out.dtype != self.out_dtype
                                or not out.is_contiguous() or out.device != self.device):
            raise ValueError(f"out must be a contiguous {self.out_dtype} ({self.n_streams}, {self.E}) tensor")
        y = out if out is not None else torch.empty((self.n_streams, self.E), dtype=self.out_dtype, device=self.device)
        r = C.c_int()
        check(lib().co_mha_step(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), int(update_state),
                                C.byref(r), _stream(stream)))
        return y if r.value else None

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """Batch mode: x (B, E, T) -> (B, E, T) with T == window (SPEC S:370-372:
        the fixed-window form, whose last column is the step output)."""
        B, E, T = x.shape
        if T != self.window:
            raise ValueError(f"batch attention needs T == window ({T} != {self.window})")
        xt = x.transpose(1, 2).contiguous().to(torch.bfloat16)           # (B, T, E)
        y = torch.empty((B, T, E), dtype=self.out_dtype, device=self.device)
        check(lib().co_mha_forward(self._h, C.c_void_p(xt.data_ptr()), T, C.c_void_p(y.data_ptr()), _stream(stream)))
        return y.transpose(1, 2)

    def clean_state(self, stream=None):
        check(lib().co_mha_clean(self._h, _stream(stream)))

    def state_dict_stream(self, stream=None):
        """(state (window-1, 2, B, E) bf16: keys then values, oldest first; n)."""
        nb = C.c_size_t()
        check(lib().co_mha_state_bytes(self._h, C.byref(nb)))
        st = torch.empty((self.window - 1, 2, self.n_streams, self.E), dtype=torch.bfloat16, device=self.device)
        n = C.c_int64()
        check(lib().co_mha_state_get(self._h, C.c_void_p(st.data_ptr()) if st.numel() else None, nb.value,
                                     C.byref(n), _stream(stream)))
        return st, n.value

    def load_state_stream(self, state: torch.Tensor, n: int, stream=None):
        nb = C.c_size_t()
        check(lib().co_mha_state_bytes(self._h, C.byref(nb)))
        state = state.to(torch.bfloat16).contiguous()
        check(lib().co_mha_state_set(self._h, C.c_void_p(state.data_ptr()) if state.numel() else None, nb.value,
                                     n, _stream(stream)))


class Stack:
    """Sequential continual network: Empty short-circuits."""

    def __init__(self, layers: Sequence[Conv]):
        self.layers = list(layers)
        arr = (C.c_void_p * len(layers))(*[l._h.value for l in layers])
        h = C.c_void_p()
        check(lib().co_stack_create(arr, len(layers), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().co_stack_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def delay(self) -> int:
        d = C.c_int64()
        check(lib().co_stack_delay(self._h, C.byref(d)))
        return d.value

    def forward_step(self, x: Optional[torch.Tensor], update_state: bool = True, out: Optional[torch.Tensor] = None,
                     stream=None) -> Optional[torch.Tensor]:
        if x is None:                                  # Empty input: nothing advances
            return None
        self.layers[0]._check_in(x, clip=False)
        last = self.layers[-1]
        shape = (last.n_streams, last.out_channels) + last.out_spatial
        if out is not None:
            last._check_out(out, shape, last.out_dtype)
        y = out if out is not None else _empty_cl(shape, last.out_dtype, last.device)
        r = C.c_int()
        check(lib().co_stack_step(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), int(update_state),
                                  C.byref(r), _stream(stream)))
        return y if r.value else None

    def forward_step_host(self, x_host: torch.Tensor, y_host: torch.Tensor, update_state: bool = True,
                          stream=None) -> bool:
        """One tick with host (pinned) buffers: x_host (B, *S, Cin), y_host
        (B, *S', Cout) channels-last; synchronises the stream."""
        r = C.c_int()
        check(lib().co_stack_step_host(self._h, C.c_void_p(x_host.data_ptr()), C.c_void_p(y_host.data_ptr()),
                                       int(update_state), C.byref(r), _stream(stream)))
        return bool(r.value)

    def forward_steps_host(self, x_host: torch.Tensor, y_host: torch.Tensor, stream=None):
        """co_stack_steps_host: (n_ready, ready_mask)."""
        return _steps_host(lib().co_stack_steps_host, self._h, x_host, y_host, stream)

    def clean_state(self, stream=None):
        check(lib().co_stack_clean(self._h, _stream(stream)))

    @property
    def graph_period(self) -> int:
        """co_stack_graph_period: a steady-state graph of a multiple of this many
        ticks replays indefinitely."""
        p = C.c_int64()
        check(lib().co_stack_graph_period(self._h, C.byref(p)))
        return p.value

    def capture(self, xs: Sequence[torch.Tensor], ys: Sequence[torch.Tensor]) -> "Graph":
        """co_stack_graph_create: record the next len(xs) ticks (frame xs[t] in,
        the Ready output to ys[t]) as one CUDA graph; clocks do not move until
        Graph.launch() replays them."""
        if len(xs) != len(ys) or not xs:
            raise ValueError("need one output buffer per frame")
        last = self.layers[-1]
        shape = (last.n_streams, last.out_channels) + last.out_spatial
        for x in xs:
            self.layers[0]._check_in(x, clip=False)
        for y in ys:
            last._check_out(y, shape, last.out_dtype)
        n = len(xs)
        xa = (C.c_void_p * n)(*[x.data_ptr() for x in xs])
        ya = (C.c_void_p * n)(*[y.data_ptr() for y in ys])
        h = C.c_void_p()
        check(lib().co_stack_graph_create(self._h, n, xa, ya, C.byref(h)))
        return Graph(h, self, list(xs), list(ys))

    def clean_streams(self, streams, stream=None):
        """Restart the given streams (indices or bool mask): layer 0 now, each
        later layer when the stream's first valid input reaches it."""
        m = _stream_mask(streams, self.layers[0].n_streams)
        check(lib().co_stack_clean_streams(self._h, m, _stream(stream)))

    def stream_ready(self) -> torch.Tensor:
        """Per-stream readiness (bool, B) of the stack's last step."""
        B = self.layers[-1].n_streams
        m = (C.c_uint8 * B)()
        check(lib().co_stack_stream_ready(self._h, m))
        return torch.tensor(list(m), dtype=torch.bool)


class Graph:
    """A captured run of stack ticks (co_graph): ``launch()`` replays them as
    the stack's next ticks and returns how many were Ready."""

    def __init__(self, h, stack: "Stack", xs, ys):
        self._h, self.stack, self._keep = h, stack, (xs, ys)   # the graph holds these pointers

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().co_graph_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def n_ticks(self) -> int:
        n, p = C.c_int64(), C.c_int()
        check(lib().co_graph_info(self._h, C.byref(n), C.byref(p)))
        return n.value

    @property
    def pdl(self) -> bool:
        n, p = C.c_int64(), C.c_int()
        check(lib().co_graph_info(self._h, C.byref(n), C.byref(p)))
        return bool(p.value)

    def upload(self, stream=None):
        check(lib().co_graph_upload(self._h, _stream(stream)))

    def launch(self, stream=None) -> int:
        nr = C.c_int64()
        check(lib().co_graph_launch(self._h, C.byref(nr), _stream(stream)))
        return nr.value
