/*
 * co_oracle.h — plain, slow, obviously-correct fp64 CPU oracle for the
 * continual-convolution step of Continual Inference Networks (arXiv 2204.03418).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2204_03418_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b, "S:a-b" = SPEC.md.
 * Every function names the passage it follows.  Readings of gaps in the paper
 * are listed in DESIGN.md ("Readings" table, A1..A20).
 *
 * Layouts (Assumption 1): every array is fp64, C order, with the
 * paper's dimension order:
 *   step  x : (B, Cin, S1, S2)          clip x : (B, Cin, T, S1, S2)
 *   step  y : (B, Cout, S1', S2')       clip y : (B, Cout, T', S1', S2')
 *   weight W: (Cout, Cin/groups, kt, kh, kw)   bias: (Cout) or NULL
 * Missing spatial axes (Conv1d: rank 0; Conv2d-over-time: rank 1) are size 1.
 */
#ifndef CO_ORACLE_H
#define CO_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int spatial_rank;                 /* 0: Conv1d over T; 1: (T,S1); 2: Conv3d (T,S1,S2) */
  int cin, cout, groups;
  int kernel[3], stride[3], padding[3], dilation[3];  /* index 0 = temporal */
  int in_spatial[2];                /* S1, S2 (ignored beyond spatial_rank) */
} or_desc;

/* Derived sizes. Return 0 on success, -1 on an invalid descriptor. */
int  or_validate(const or_desc* d);
int  or_receptive_field(const or_desc* d);          /* f = dil_t (kt-1) + 1 */
int  or_delay(const or_desc* d);                    /* P:138-145  d = f - p - 1 */
int  or_out_spatial(const or_desc* d, int out[2]);  /* S1', S2' */
int  or_out_len(const or_desc* d, int T);           /* S:64 T' = floor((T+2p-f)/s)+1 (may be < 1) */
int  or_ring_slots(const or_desc* d);               /* R = ceil((f-1)/s): outputs pending at once */

/* O1 (Definition 1; S:241 cross-correlation): one output value of the
 * regular convolution for stream-local frames Z[0..kt-1], each a (Cin,S1,S2)
 * array given by a base pointer and strides (element units); Z[k].p == NULL
 * means an all-zero (padded or not-yet-seen) frame.  bias may be NULL. */
typedef struct { const double* p; long sc, sh, sw; } or_frame;
double or_column_at(const or_desc* d, const double* W, const double* bias,
                    const or_frame* Z, int o, int ho, int wo);
/* O1 over all outputs of one stream: y[o*y_sc + ho*S2' + wo]. */
void   or_column(const or_desc* d, const double* W, const double* bias,
                 const or_frame* Z, double* y, long y_sc);

/* O2 ("operates identically to forward"): batch forward over a
 * clip, temporal zero padding p at both ends.  Returns T' or -1 if T' < 1. */
int or_forward(const or_desc* d, const double* W, const double* bias,
               int B, const double* x, int T, double* y);

/* O3: the step machine.  Keeps the last f-1 padded
 * input frames (start padding = zero frames already in the history).
 * Ready iff n >= d and (n-d) mod s == 0.  On Ready, the output is
 * the batch column (n-d)/s computed from the window (O1). */
typedef struct or_step or_step;
or_step* or_step_new(const or_desc* d, const double* W, const double* bias, int B);
void     or_step_free(or_step* sm);
void     or_step_clean(or_step* sm);                  /* P:116 clean_state() */
long     or_step_count(const or_step* sm);            /* n: stateful steps since clean */
/* x: (B,Cin,S1,S2) or NULL for an all-zero frame (pad_end).  y: (B,Cout,S1',S2').
 * Returns ready (1) / Empty (0); y untouched on Empty. */
int      or_step_forward(or_step* sm, const double* x, int update_state, double* y);
/* head = ceil((n-d)/s) mod R (floored mod): the slot index of the next output
 * to complete in the GPU ring convention (A20); reported for bit-exact checks. */
int      or_step_head(const or_step* sm);

/* O4: fold of or_step_forward over the T columns of a clip,
 * then p zero steps if pad_end.  ready_mask has T (+p) entries; y receives the
 * Ready outputs compacted in time (A1): y is (B,Cout,T(+p),S1',S2') and its
 * first n_ready time entries are written.  Returns n_ready. */
int or_step_forward_steps(or_step* sm, const double* x, int T, int pad_end,
                          int update_state, uint8_t* ready_mask, double* y);

/* O5 (A8, A9, A20): canonical state.  R slots; slot j holds output
 * i_next + j where i_next = ceil((n-d)/s) is the next output to complete.  Its
 * value is the sum of the contributions of the frames consumed so far
 * (start padding included as zeros), bias excluded; outputs i < 0 (never
 * emitted) are 0.  Layout (R, B, Cout, S1', S2'). */
void or_step_state(const or_step* sm, double* state);
/* Raw history: the last f-1 padded frames, oldest first, (f-1, B, Cin, S1, S2). */
void or_step_history(const or_step* sm, double* out);

/* O7: brute-force sliding window.  hist holds every real frame fed
 * so far, (B,Cin,n+1,S1,S2) with n+1 frames (x_0..x_n).  Re-runs O2 with no
 * padding over [p zeros | x_0..x_n] and returns the column of tick n when
 * tick n is Ready (returns 1), else 0. */
int or_bruteforce_tick(const or_desc* d, const double* W, const double* bias,
                       int B, const double* hist, int n_plus_1, double* y);

/* O6: sequential stack of step machines.
 * Empty short-circuits the downstream layers without advancing them (A7).
 * After each layer: + bias (inside O1), optional ReLU, optional bf16 RNE
 * rounding (the build's declared quantisation points, A16/A17). */
typedef struct or_stack or_stack;
or_stack* or_stack_new(int n_layers, const or_desc* descs, const double* const* Ws,
                       const double* const* biases, const int* relu, const int* round_bf16,
                       int B);
void or_stack_free(or_stack* st);
void or_stack_clean(or_stack* st);
/* Returns 1 if the last layer emitted (y written), else 0. */
int  or_stack_forward(or_stack* st, const double* x, int update_state, double* y);

/* Principle 5 / 6 in the worked-example reading (A3):
 * s_acc(i) = s(i) s_acc(i-1); p_acc(i) = p_acc(i-1) + p(i) s_acc(i-1);
 * f_acc(i) = f_acc(i-1) + (f(i)-1) s_acc(i-1); d_acc = f_acc - p_acc - 1. */
void or_accumulate(int n, const int* f, const int* p, const int* s,
                   int* s_acc, int* p_acc, int* f_acc, int* d_acc);
/* Readiness schedule: tick t is Ready iff t >= d and (t-d) mod s == 0. */
int  or_schedule_ready(int d_nn, int s_nn, long t);

/* Round an fp64 value to the nearest bfloat16 (8 significant bits), ties to
 * even (A17).  Used only for the stack's declared quantisation points. */
double or_bf16_round(double x);
void   or_bf16_round_array(double* x, long n);

/* Analytic cost model (1 MAC = 2 FLOP), per stream-step. */
double or_flops_step(const or_desc* d);

#ifdef __cplusplus
}
#endif
#endif
