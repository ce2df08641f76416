/*
 * co.h — C ABI of the B200-native continual-convolution step
 * (Continual Inference Networks, arXiv 2204.03418).
 *
 * Citations: "P:a-b" = PAPER.md lines a-b (/root/reference), "S:a-b" = SPEC.md.
 *
 * What the library computes (the hot path of BASELINE.json's north_star):
 *   a continual 3D / 2D / 1D convolution layer (co.Conv3d, co.Conv1d)
 *   run for n_streams independent streams that share one clock.  Each
 *   co_forward_step convolves one incoming frame with every temporal slice of
 *   the kernel ("compute inputs step-by-step"), adds the partial sums into
 *   a per-stream fp32 ring of pending outputs, emits the output whose receptive
 *   field is complete (or reports Empty while n < delay), and
 *   rotates the ring.  The emitted value equals the matching column of the
 *   regular convolution (Definition 1).
 *
 * Conventions shared by every call
 *  - Return value: CO_OK (0) or a negative co_status.  Nothing aborts, no C++
 *    exception crosses the ABI; co_last_error() returns a thread-local message
 *    for the last failing call on this thread.
 *  - Pointers are DEVICE pointers unless the parameter says "host".
 *  - Asynchrony: device work is enqueued on the caller's CUDA stream
 *    (`co_stream` = cudaStream_t; NULL = legacy default stream) and calls
 *    return after enqueue.  Host outputs (ready, ready_mask, n_ready, T_out,
 *    info) are final on return because the clock lives on the host (a1).  No
 *    call synchronises the device except the *_host variants, so step loops are
 *    CUDA-graph capturable.
 *  - Concurrency: a handle has a single writer; different handles
 *    may run concurrently on different streams.  co_forward only reads the
 *    packed weights and may overlap other calls on the same handle.
 *  - Layout (Assumption 1): tensors keep the paper's LOGICAL order
 *    (B, C, S1, S2) per step and (B, C, T, S1, S2) per clip, stored
 *    CHANNELS-LAST: step memory is (B, S1, S2, C), clip memory is
 *    (B, T, S1, S2, C), dense.  (PyTorch: torch.channels_last /
 *    torch.channels_last_3d.)  Absent spatial axes have extent 1.
 *  - Weights: (Cout, Cin/groups, kt, kh, kw) dense, in w_dtype (PyTorch's
 *    Conv weight layout, Principle 1 P:71-80); bias: (Cout) fp32 or NULL.  The
 *    library never rounds weights: they arrive already in w_dtype.
 *  - Arithmetic: products in fp32 (bf16 x bf16 is exact in fp32), sums in
 *    fp32, state in fp32; outputs rounded to out_dtype with round-to-nearest-even.
 */
#ifndef CO_H
#define CO_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define CO_ABI_VERSION 4
#define CO_MAX_KT 32          /* temporal kernel extent supported by the kernels */

typedef enum {
  CO_OK = 0,
  CO_ERR_ARG = -1,          /* bad descriptor / argument (e.g. p_t > f-1; groups not dividing channels) */
  CO_ERR_SHAPE = -2,        /* shape, byte-count or meta mismatch; layer chaining in a stack */
  CO_ERR_LENGTH = -3,       /* co_forward with T' < 1 */
  CO_ERR_UNSUPPORTED = -4,  /* no sm_100a kernel for this combination (there is no CPU fallback) */
  CO_ERR_CUDA = -5,         /* a CUDA runtime/driver error; message carries cudaGetErrorString */
  CO_ERR_OOM = -6           /* device allocation failed */
} co_status;

typedef enum { CO_F32 = 0, CO_BF16 = 1 } co_dtype;
typedef enum { CO_ACT_NONE = 0, CO_ACT_RELU = 1 } co_activation;
/* Kernel family for the step (SURVEY §8a dispatch rule).  AUTO picks by shape. */
typedef enum {
  CO_KERNEL_AUTO = 0,
  CO_KERNEL_DIRECT = 1,     /* generic CUDA-core kernel: any groups/dilation/stride, fp32 or bf16 */
  CO_KERNEL_DENSE_TC = 2,   /* tcgen05/TMEM implicit GEMM with fused state epilogue (bf16, dense) */
  CO_KERNEL_DEPTHWISE = 3,  /* CUDA-core depthwise stencil (groups == Cin == Cout, bf16) */
  CO_KERNEL_POOL = 4,       /* CUDA-core window max / mean over the RAW ring (pooling handles only) */
  CO_KERNEL_COPY = 5        /* ring copies only (Delay handles) */
} co_kernel;

/* Per-stream state layout (BASELINE.json north_star "Per-stream state layout";
 * SURVEY §8f row f1).  PSUM: the fp32 ring of R pending partial sums (each frame
 * contracted with all kt slices once, 2(kt-1) fp32 state accesses per output).
 * RAW: a ring of the last f input frames in the input dtype (SPEC's layout,
 * S:227); a Ready step contracts the whole window (K = kt kh kw Cin/g),
 * a non-Ready step only stores its frame.  Same outputs (Definition 1). */
typedef enum { CO_STATE_PSUM = 0, CO_STATE_RAW = 1, CO_STATE_AUTO = 2 } co_state_layout;
/* AUTO: the planner picks per layer -- RAW for bf16 dense layers with a 1x1
 * spatial kernel (the flat tensor-core RAW kernel) when the RAW ring moves at
 * most half the bytes of the fp32 partial sums per step (kt+1 frames vs
 * 2 (kt-1) fp32 output slots), PSUM otherwise; co_conv_info reports the
 * choice.  Use PSUM where a workload mandates fp32 state. */

/* Operation of a handle ("Pooling:
 * co.AvgPool1d, co.MaxPool1d, etc.").  A pooling handle has
 * in_channels == out_channels (groups is ignored), no weights or bias
 * (create takes weights = bias = NULL), dispatches CO_KERNEL_POOL, and keeps a
 * ring of the last f SPATIALLY REDUCED frames (B, S1', S2', C): pooling is
 * separable, so each step reduces its frame over the spatial window once and a
 * Ready step folds kt reduced frames (state_layout is ignored; co_info reports
 * RAW).  kt is not bounded by CO_MAX_KT (the paper's 64-step expanded global
 * average pooling).  Padding (temporal and spatial) is 0 and counted in
 * the divisor for AVG (count_include_pad, divisor kt kh kw, A21) and
 * is ignored for MAX (PyTorch's implicit -inf padding; a window of padding only
 * yields -inf, A22).  Canonical state (co_state_get): (f-1, B, S1', S2', C),
 * MAX in in_dtype with padded frames -inf, AVG fp32 spatial-window sums with
 * padded frames 0.  Clock, readiness, delay and the call modes are those of a
 * convolution with the same kernel / stride / padding / dilation
 * (Definition 1). */
typedef enum { CO_OP_CONV = 0, CO_OP_MAX_POOL = 1, CO_OP_AVG_POOL = 2, CO_OP_DELAY = 3 } co_op;
/* CO_OP_DELAY (co.Delay): kernel[0] = d + 1 (so f = d + 1,
 * delay d), every other kernel / stride / dilation entry 1, padding 0,
 * in_channels == out_channels, out_dtype == in_dtype, no weights or bias.  A
 * step emits Empty while n < d, then the input of d ticks ago (a copy out of a
 * ring of d + 1 frames, CO_KERNEL_COPY); batch mode (co_forward) is the
 * identity on the clip (T' = T).  Canonical state: the last d frames,
 * (d, B, S1, S2, C) in in_dtype. */

typedef void* co_stream;                 /* cudaStream_t */
typedef struct co_conv co_conv;          /* opaque: packed weights, fp32 state ring, host clock */
typedef struct co_stack co_stack;        /* opaque: ordered layers + inter-layer activations */

/* Layer descriptor.  Index 0 of kernel/stride/padding/dilation is temporal
 * (kernel[0] = kt, padding[0] = temporal padding p).  Entries beyond
 * spatial_rank are ignored (treated as 1 / 0). */
typedef struct {
  int32_t spatial_rank;                  /* 0: Conv1d over T; 1: (T,S1); 2: Conv3d (T,S1,S2) */
  int32_t in_channels, out_channels, groups;
  int32_t kernel[3], stride[3], padding[3], dilation[3];
  int32_t in_spatial[2];                 /* S1, S2 of one step */
  int64_t n_streams;                     /* B: independent streams, one shared clock */
  int32_t in_dtype;                      /* co_dtype of x */
  int32_t w_dtype;                       /* co_dtype of weights (must equal in_dtype) */
  int32_t out_dtype;                     /* co_dtype of y */
  int32_t activation;                    /* co_activation applied to emitted outputs (after bias) */
  int32_t kernel_choice;                 /* co_kernel; AUTO = dispatch rule */
  int32_t state_layout;                  /* co_state_layout (PSUM = 0 default) */
  int32_t op;                            /* co_op (CONV = 0 default) */
} co_conv_desc;

/* Clock + geometry of a handle.  n and head are the host clock (a1). */
typedef struct {
  int64_t n;                 /* stateful steps since clean */
  int32_t head;              /* ceil((n-d)/s) mod R, floored mod: ring slot of the next output to complete */
  int32_t ring_slots;        /* R = ceil((f-1)/s) pending outputs (0 when f = 1) */
  int32_t delay;             /* d = f - p - 1 */
  int32_t receptive_field;   /* f = dil_t (kt-1) + 1 */
  int32_t stride_t;          /* s */
  int32_t padding_t;         /* p */
  int32_t out_spatial[2];    /* S1', S2' */
  int32_t kernel_used;       /* co_kernel actually dispatched */
  int32_t state_layout;      /* co_state_layout of the handle */
} co_info;

/* ---- lifetime ------------------------------------------------------------ */

/* Create a layer: the co.Conv constructor of Listing 1 with the
 * nn.Conv arguments it extends (Principle 1: identical / extended
 * constructors, identical weights -- the (Cout, Cin/g, kt, kh, kw) tensor of
 * nn.Conv3d, so a regular layer's state_dict loads unchanged).
 * `weights` (Cout, Cin/g, kt, kh, kw) in w_dtype and `bias`
 * (Cout, fp32, may be NULL) are host pointers if weights_on_device == 0, else
 * device pointers; both are copied and repacked, so the caller may free them on
 * return.  The fp32 state (R slots x B x S1' x S2' x Cout) is allocated and
 * zeroed (clean state, A8).  Errors: CO_ERR_ARG, CO_ERR_UNSUPPORTED, CO_ERR_OOM,
 * CO_ERR_CUDA.  Synchronises the current device once (setup, not the hot path). */
int co_conv_create(const co_conv_desc* desc, const void* weights, const float* bias,
                   int weights_on_device, co_conv** out);
int co_conv_destroy(co_conv* h);                      /* frees weights, state, clock; NULL ok (no paper
                                                         passage: the C ABI's ownership rule) */
int co_conv_info(const co_conv* h, co_info* info);    /* host, final on return */
int co_delay(const co_conv* h, int64_t* delay);       /* d = f - p - 1 */
const char* co_kernel_name(const co_conv* h);         /* name of the dispatched step kernel */

/* ---- call modes (Principle 2) ----------------------------------- */

/* forward_step: x one step (B, S1, S2, Cin) channels-last in in_dtype;
 * y (B, S1', S2', Cout) in out_dtype.  *ready (host) = 1 when the output is
 * emitted (n >= d and (n-d) mod s == 0), else 0 (Empty) and y is left
 * untouched.  x == NULL feeds an all-zero step (used for pad_end; a padding
 * step, -inf, for MAX pooling handles).  With
 * update_state == 0 the ready output is computed from the current state and
 * state + clock stay bitwise unchanged. */
int co_forward_step(co_conv* h, const void* x, void* y, int update_state, int* ready, co_stream stream);

/* Same step with HOST buffers: x_host / y_host are host memory (pinned for
 * best speed); the call copies x in, runs the step, copies y out and
 * synchronises `stream` before returning, so y_host is valid on return. */
int co_forward_step_host(co_conv* h, const void* x_host, void* y_host, int update_state, int* ready,
                         co_stream stream);

/* Streaming with HOST buffers: T frames, TIME-major on the host, x_host
 * (T, B, S1, S2, Cin) pinned memory (frame t of all streams contiguous, the
 * order frames arrive in online inference); the Ready outputs are written
 * compacted to y_host (n_ready, B, S1', S2', Cout).  The H2D copy of frame t+1
 * and the D2H copy of output t-1 overlap step t (double-buffered device
 * staging, two extra internal streams); state updates as co_forward_step with
 * update_state = 1.  Synchronises `stream` before returning: y_host, ready_mask
 * (host, may be NULL, T flags) and *n_ready are final on return. */
int co_forward_steps_host(co_conv* h, const void* x_host, int64_t T, void* y_host, uint8_t* ready_mask,
                          int64_t* n_ready, co_stream stream);

/* forward_steps: the fold of co_forward_step over the T columns of the
 * clip x (B, T, S1, S2, Cin), then p zero steps if pad_end.  y receives
 * the Ready outputs compacted in time (A1): (B, n_ready, S1', S2', Cout); its
 * capacity must be co_steps_ready_count(h, T, pad_end) columns.  ready_mask
 * (host, may be NULL) gets T + (pad_end ? p : 0) flags; *n_ready (host).
 * Bitwise equal to the fold of co_forward_step.  With update_state == 0
 * the fold runs on a device copy of the state. */
int co_forward_steps(co_conv* h, const void* x, int64_t T, void* y, uint8_t* ready_mask,
                     int64_t* n_ready, int pad_end, int update_state, co_stream stream);
/* Number of Ready ticks the next co_forward_steps(T, pad_end) will produce. */
int co_steps_ready_count(const co_conv* h, int64_t T, int pad_end, int64_t* n_ready);

/* forward: batch mode, x (B, T, S1, S2, Cin) -> y (B, T', S1', S2',
 * Cout) with symmetric temporal zero padding p and T' = floor((T+2p-f)/s)+1
 * (S:64).  Neither reads nor writes state.  CO_ERR_LENGTH if T' < 1. */
int co_forward(co_conv* h, const void* x, int64_t T, void* y, int64_t* T_out, co_stream stream);
int co_forward_out_len(const co_conv* h, int64_t T, int64_t* T_out);

/* ---- state (Principle 3) -------------------------------------- */

/* Canonical state, PSUM layout: fp32 (R, B, S1', S2', Cout) dense, device memory.
 * Slot j holds output i_next + j, i_next = ceil((n-d)/s) the next output to
 * complete; its value is the sum of contributions of the frames consumed so far
 * (bias excluded, A9), 0 for outputs that are never emitted (i < 0).
 * RAW layout: in_dtype (f-1, B, S1, S2, Cin): slot j holds padded frame
 * m-(f-1)+j, m = n + p the next frame's padded index (oldest first; the start
 * padding is zero).  `bytes` must equal co_state_bytes().  get fills *meta with the clock; set restores the
 * clock from *meta (its geometry fields must match: CO_ERR_SHAPE).  A get ->
 * set round trip is bitwise (checkpoint / resume). */
/* co_state_bytes: the size of the module's internal state (the buffers P:110-116
 * step, clean with clean_state() and skip with update_state=False) in the
 * canonical layout above. */
int co_state_bytes(const co_conv* h, size_t* bytes);
int co_state_get(co_conv* h, void* dst, size_t bytes, co_info* meta, co_stream stream);
int co_state_set(co_conv* h, const void* src, size_t bytes, const co_info* meta, co_stream stream);
/* clean_state(): zero state, n = 0. */
int co_state_clean(co_conv* h, co_stream stream);

/* ---- layer stack (Sequential; Principle 6 P:248-264) -------- */

/* Chain layers: layer i's output geometry/dtype must equal layer i+1's input
 * (CO_ERR_SHAPE otherwise) and all layers share n_streams.  The stack owns its
 * inter-layer activation buffers, not its layers.  Each step threads the frame
 * through the layers; an Empty output ends the tick and the downstream layers
 * are not advanced (A7). */
int co_stack_create(co_conv* const* layers, int n_layers, co_stack** out);
int co_stack_destroy(co_stack* st);
int co_stack_step(co_stack* st, const void* x, void* y, int update_state, int* ready, co_stream stream);
/* Same tick with HOST buffers (first layer's input, last layer's output):
 * copies x_host in, runs the tick, copies y_host out if Ready, synchronises
 * `stream`; y_host is valid on return. */
int co_stack_step_host(co_stack* st, const void* x_host, void* y_host, int update_state, int* ready,
                       co_stream stream);
/* co_forward_steps_host for a stack: time-major host frames of layer 0 in, the
 * last layer's Ready outputs (compacted) out, copies overlapped with the ticks. */
int co_stack_steps_host(co_stack* st, const void* x_host, int64_t T, void* y_host, uint8_t* ready_mask,
                        int64_t* n_ready, co_stream stream);
/* Accumulated delay d_NN (Principle 6 in the worked-example reading, A3). */
int co_stack_delay(const co_stack* st, int64_t* d_nn);
int co_stack_clean(co_stack* st, co_stream stream);

/* ---- CUDA-graph step loops ---------------------------------------------------- */

/* A stack's tick schedule is a function of the host clocks alone (readiness
 * n >= d and (n-d) mod s == 0; ring slots from n, the a1/a5
 * rows), so a run of ticks can be captured once into a CUDA graph and
 * replayed with one launch -- no per-tick host work or launch latency, which
 * is what small stream shards are bound by.
 * co_stack_graph_create records the next n_ticks ticks of `st` (update_state =
 * 1) from the current clocks, tick t reading the device frame x[t] (host array
 * of n_ticks device pointers, layer 0's input layout) and writing the last
 * layer's Ready output to y[t] (device pointers, may repeat); nothing executes
 * and no clock moves.  co_graph_launch enqueues the recorded ticks on `stream`
 * and advances every layer's clock by n_ticks (*n_ready, host, = the ticks on
 * which the stack was Ready).  It refuses with CO_ERR_ARG unless every layer's
 * clock is where the recorded schedule starts: the same n, or, once all
 * transients are past (n >= f + p + d + 2s), the same phase modulo a period of
 * every clock-derived kernel argument -- so in steady state a graph of any
 * multiple of that period replays indefinitely, and outputs equal the eager
 * fold of co_stack_step bit for bit.  Also CO_ERR_ARG if a layer's internal
 * staging moved since capture, CO_ERR_UNSUPPORTED while a per-stream clean
 * (co_stack_clean_streams) is still pending.  The graph keeps pointers to the
 * stack, its layers and x / y: they must outlive it.  Programmatic dependent
 * launch edges are captured when the driver instantiates them (co_graph_info
 * reports pdl = 1), else the graph uses plain launches. */
typedef struct co_graph co_graph;
int co_stack_graph_create(co_stack* st, int64_t n_ticks, const void* const* x, void* const* y, co_graph** out);
int co_graph_upload(co_graph* g, co_stream stream);      /* optional: pre-upload before the first launch */
/* The stack's schedule period in ticks: in steady state a graph of any
 * multiple of it returns every layer to its captured phase (replays forever). */
int co_stack_graph_period(const co_stack* st, int64_t* period);
int co_graph_launch(co_graph* g, int64_t* n_ready, co_stream stream);
int co_graph_info(const co_graph* g, int64_t* n_ticks, int* pdl);
int co_graph_destroy(co_graph* g);

/* ---- composition: BroadcastReduce ------------------------ */

/* BroadcastReduce(branches, reduce) (Listing 3
 * "co.BroadcastReduce(conv, co.Delay(1))", Listing 4 reduce="concat";
 * Principle 7 P:280-288): the input step is broadcast to
 * every branch -- a co_stack (owned by the caller, used by this composite only)
 * or NULL for the identity -- and the branch outputs are merged.  Branches keep
 * the frame rate (accumulated temporal stride 1) and share the output spatial
 * shape; stack branches share the output dtype (the composite's); for SUM the
 * channel count is common and an identity branch in another dtype is added
 * with conversion; CONCAT needs one dtype.  A branch with delay d_i < d_max is suffixed with Delay(d_max - d_i)
 * on its Ready outputs (a ring of d_max - d_i + 1 output frames), so the
 * composite's delay is d_max and it is Ready when every aligned branch is.
 * CONCAT stacks the channels in branch order.  Batch mode merges the first
 * T_min output columns of every branch (the columns the delay alignment pairs;
 * DESIGN.md A24). */
typedef enum { CO_REDUCE_SUM = 0, CO_REDUCE_CONCAT = 1 } co_reduce;
typedef struct co_parallel co_parallel;
int co_parallel_create(co_stack* const* branches, int n_branches, int reduce, co_parallel** out);
int co_parallel_destroy(co_parallel* p);               /* frees the composite, not the branch stacks */
int co_parallel_step(co_parallel* p, const void* x, void* y, int update_state, int* ready, co_stream stream);
int co_parallel_forward(co_parallel* p, const void* x, int64_t T, void* y, int64_t* T_out, co_stream stream);
int co_parallel_clean(co_parallel* p, co_stream stream);
int co_parallel_delay(const co_parallel* p, int64_t* delay);
/* Output geometry: channels (sum: the common count; concat: the total). */
int co_parallel_out_channels(const co_parallel* p, int32_t* channels);

/* ---- continual single-output multi-head attention -------- */

/* co.MultiheadAttention in "single-output" mode (SPEC.md:
 * 357-403) over n_streams lockstep streams: each step projects x_t (B, E) to
 * q, k, v, pushes (k, v) into a ring of `window` = n entries and, once n
 * entries are present (delay d = n - 1, stride 1; no early partial windows,
 * S:392), emits the attention of the newest query against the n keys / values
 * (per head softmax(q k^T / sqrt(E / heads)) v, heads concatenated) projected
 * by W_o -- the last column of batch attention over the trailing n steps.
 * Weights in PyTorch's nn.MultiheadAttention layout: w_qkv (3E, E) = [W_q; W_k;
 * W_v], w_o (E, E), bf16; biases fp32 (3E) / (E), may be NULL; host pointers
 * unless weights_on_device.  x, y bf16 (y fp32 if out_dtype = CO_F32).  Head
 * dims 32, 64 or 128.  Canonical state: the last n-1 keys and values,
 * (n-1, 2, B, E) bf16 (k then v per slot, oldest first). */
typedef struct {
  int32_t embed_dim, num_heads, window;
  int64_t n_streams;
  int32_t out_dtype;                     /* co_dtype of y */
} co_mha_desc;
typedef struct co_mha co_mha;
int co_mha_create(const co_mha_desc* d, const void* w_qkv, const float* b_qkv, const void* w_o, const float* b_o,
                  int weights_on_device, co_mha** out);
int co_mha_destroy(co_mha* m);
int co_mha_step(co_mha* m, const void* x, void* y, int update_state, int* ready, co_stream stream);
/* Batch mode: x (B, T, E) -> y (B, T, E), full attention over the T columns;
 * T must equal window (the fixed-window form; its last column is
 * the step output): CO_ERR_LENGTH otherwise.  Neither reads nor writes state;
 * stream-ordered temporaries. */
int co_mha_forward(co_mha* m, const void* x, int64_t T, void* y, co_stream stream);
int co_mha_clean(co_mha* m, co_stream stream);
int co_mha_delay(const co_mha* m, int64_t* delay);
int co_mha_state_bytes(const co_mha* m, size_t* bytes);
int co_mha_state_get(co_mha* m, void* dst, size_t bytes, int64_t* n, co_stream stream);
int co_mha_state_set(co_mha* m, const void* src, size_t bytes, int64_t n, co_stream stream);

/* ---- per-stream clocks --------- */

/* Streams join and leave independently.  A handle keeps one clock n (A19,
 * P:283 "the same global clock"); stream b's own step count is n_b = n - join_b.
 * co_state_clean_streams resets the state slices of the streams with
 * mask[b] != 0 (host array of B flags) to the clean state (zero partial sums /
 * frames; -inf for MAX pooling) and sets join_b = n; from then on stream b
 * behaves as a fresh stream whose first frame is the next step's.  Under
 * temporal stride s it must be called at n = 0 mod s (else CO_ERR_ARG), so the
 * stream's Ready phase matches the handle's.  co_state_clean and co_state_set
 * reset every join_b to 0.  Stream-ordered on `stream`. */
int co_state_clean_streams(co_conv* h, const uint8_t* mask, co_stream stream);
/* Per-stream readiness of the last step on the handle's clock (host array of B
 * flags): ready[b] = the step was Ready and n_b >= d at that step. */
int co_stream_ready(const co_conv* h, uint8_t* ready);
/* Stack form: layer 0 is cleaned now; each later layer cleans stream b when
 * its first valid input for b arrives (the layer below reports b ready), so
 * every layer sees the fresh stream from its own first frame.  Later layers
 * must have temporal stride 1 (else CO_ERR_UNSUPPORTED). */
int co_stack_clean_streams(co_stack* st, const uint8_t* mask, co_stream stream);
/* Per-stream readiness of the stack's last step (all 0 when it was Empty). */
int co_stack_stream_ready(const co_stack* st, uint8_t* ready);

/* ---- composition: Residual ------------------------------- */

/* Residual(body) with Sum ("Residual connections", Listing 3
 * P:482-504 co.Residual / residual_shrink; Principle 7 P:280-288; SPEC.md:
 * 452-458).  `body` is a sequence of layer handles (owned by the caller, not
 * shared with another stack or residual, alive until co_residual_destroy) run
 * as a stack; it must keep the frame rate (accumulated temporal stride 1), the
 * channel count, spatial shape and dtype of its input (body[0] in_dtype ==
 * body[n-1] out_dtype).  Alignment of the identity branch ("centered",
 * P:312-316):
 *  shrink = 0: equal padding, 2 p_acc = f_acc - 1; the identity branch is
 *              delayed by the body's delay d (Fig. 4); batch y = x + body(x);
 *  shrink = 1: f_acc odd (any padding with p_acc <= (f_acc-1)/2); the identity
 *              branch is delayed by (f_acc-1)/2 and, in batch mode, cropped by
 *              (f_acc-1)/2 at each end.
 * The composite's delay is the body's (the larger branch delay, Principle 7);
 * it is Ready exactly when the body is.  `activation` (co_activation) is
 * applied after the add (the ResNet / X3D block form).  The identity branch's
 * frames live in a ring of d_skip + 1 frames in the input dtype.  Errors:
 * CO_ERR_ARG, CO_ERR_SHAPE (shape / timing contract), CO_ERR_OOM. */
typedef struct co_residual co_residual;
int co_residual_create(co_conv* const* body, int n_layers, int shrink, int activation, co_residual** out);
int co_residual_destroy(co_residual* r);              /* frees the composite, not the body layers */
/* One tick (same contract as co_forward_step): x (B, S1, S2, C) channels-last,
 * y (B, S1, S2, C) in the body's out_dtype; *ready = 1 when emitted. */
int co_residual_step(co_residual* r, const void* x, void* y, int update_state, int* ready, co_stream stream);
/* Batch mode: x (B, T, S1, S2, C) -> y (B, T', S1, S2, C), T' = the body's output
 * length; neither reads nor writes state.  Temporaries are stream-ordered
 * allocations freed before return (stream order). */
int co_residual_forward(co_residual* r, const void* x, int64_t T, void* y, int64_t* T_out, co_stream stream);
int co_residual_clean(co_residual* r, co_stream stream);   /* body layers + identity ring + clock */
/* Composite delay (= the body's d_nn) and the identity branch's delay. */
int co_residual_delay(const co_residual* r, int64_t* delay, int64_t* skip_delay);

/* ---- planner / launch options ----------------------------------------------- */

/* The library reads no environment variable: these named, process-wide
 * options are its only switches.  Each selects among the sm_100a kernels or
 * launch modes; none skips work or changes a result beyond the fp32 summation
 * order (the exact-integer regime, stays bitwise).  They exist
 * so tests can drive every kernel path and A/B runs can compare launch modes;
 * the defaults are the planner's measured choices.  [create]: read by
 * co_conv_create / co_mha_create (affects handles created afterwards);
 * [launch]: read at each step launch; [call]: read by each co_forward_steps.
 *   "tc_mode"    0 auto | 1 force the tensor-core K pipeline (KLOOP)          [create]
 *   "khalo"      1 allow KHALO (default) | 0 keep the strided-gather KLOOP   [create]
 *   "pair"       0 auto | 1 single CTA | 2 CTA pairs (HALO / FLAT)            [create]
 *   "kpair"      0 auto | 1 / 2 pin the KLOOP / KHALO pairing                 [create]
 *   "eg"         0 auto | 1..4 epilogue warpgroups of the tensor-core kernel  [create]
 *   "mc"         1 (default) | 2, 4, 8 weight-multicast clusters (1-CTA KLOOP) [launch]
 *   "pdl"        1 (default) programmatic dependent launch | 0 off            [launch]
 *   "chunk"      1 (default) chunked co_forward_steps where supported | 0 fold [call]
 *   "chunk_flat" 0 (default) | 1 chunked FLAT (1x1 spatial) clips             [call]
 *   "chunk_st"   0 (default) | 1 chunked depthwise-stencil clips              [call]
 *   "chunk_t"    0 (default: up to 256) | max frames per chunked launch       [call]
 *   "pool_band"  1 (default) row-band pooling kernel | 0 plain kernel         [create]
 *   "pool_vh"   -1 auto | 0 direct fold | 1 block decomposition (pooling)     [create]
 *   "pool_g"     0 auto | 1..32 lanes per pooled output vector                [create]
 *   "log"        0 (default) | 1 print each tensor-core plan to stderr        [create]
 *   "stem"       1 (default) small-Cin stems build their W-im2col in shared
 *                memory | 0 a separate HBM W-im2col pass per step            [create]
 *   "dw_seg"     1 (default) depthwise stencils stream state + input rows
 *                through a bulk-copy stage ring (k_step_dw_seg) | 0 the
 *                per-thread-load K2 (k_step_dw_st)                           [create]
 *   "mha_ring"   1 (default) step-mode MHA attention streams each stream's
 *                K / V rings through a bulk-copy stage ring
 *                (k_mha_attend_ring, <= 16 heads) | 0 the per-lane-load
 *                kernel (k_mha_attend)                                        [launch]
 *   "pool_seg"   1 (default) bf16 pooling layers with a spatial window and a
 *                direct temporal fold stream input rows + ring rows through
 *                a bulk-copy stage ring (k_step_pool_seg) | 0 the band /
 *                plain kernels                                                [create / launch]
 * name == NULL resets every option to its default.
 * Errors: CO_ERR_ARG for an unknown name or a value out of range.  Not
 * thread-safe against concurrent creates (set options before building handles). */
int co_set_option(const char* name, int64_t value);
int co_get_option(const char* name, int64_t* value);
/* Name of option `index` (0, 1, ...), NULL past the last: lets a harness record
 * every option's value next to a measurement. */
const char* co_option_name(int index);

/* ---- misc ------------------------------------------------------------------ */
const char* co_last_error(void);   /* no paper passage: the ABI's error channel (conventions above) */
int co_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CO_H */
