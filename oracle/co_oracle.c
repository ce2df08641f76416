/*
 * co_oracle.c — fp64 CPU oracle for the continual-convolution step.
 *
 * TEST INFRASTRUCTURE ONLY (see co_oracle.h).  Plain loops, no blocking, no
 * fusion, no reordering beyond what the definitions below state, so that each
 * function can be checked against the paper by eye.  OpenMP is used only to
 * run independent streams (B) side by side; every value is computed by the
 * same sequential loop regardless of the thread count.
 *
 * Method (what is computed), with citations into /root/reference/PAPER.md:
 *  - Definition 1: step inference and batch inference produce
 *    identical outputs for identical receptive fields.  So the step output is
 *    one column of the regular (batch) convolution of the stream's history.
 *  - Principle 2: forward / forward_step / forward_steps.
 *  - Principle 3: state rules, update_state=False, clean_state().
 *  - Principle 4: delay d = f - p - 1.
 *  - Padding as delay reduction: start padding pre-saturates the
 *    state with zeros; end padding only via pad_end.
 *  - Principle 5: stride s -> Empty outputs between Ready ticks.
 *  - Principle 6 + worked example: accumulated timing (reading A3).
 *  - The continual 3D convolution itself is cited, not derived; its
 *    result is, by Definition 1, the batch column computed here (O1).
 */
#include "co_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- helpers */

/* Fill the absent spatial axes with the identity (size 1, kernel 1, stride 1,
 * padding 0, dilation 1), so every routine below can loop over (S1, S2). */
static void norm_desc(const or_desc* in, or_desc* d) {
  *d = *in;
  for (int a = 1; a <= 2; ++a) {
    if (a > d->spatial_rank) {
      d->kernel[a] = 1; d->stride[a] = 1; d->padding[a] = 0; d->dilation[a] = 1;
      d->in_spatial[a - 1] = 1;
    }
  }
}

static long floor_div(long a, long b) {          /* b > 0 */
  long q = a / b;
  if ((a % b != 0) && (a < 0)) q -= 1;
  return q;
}
static long ceil_div(long a, long b) { return -floor_div(-a, b); }
static long floor_mod(long a, long b) { return a - floor_div(a, b) * b; }

int or_validate(const or_desc* in) {
  if (!in) return -1;
  if (in->spatial_rank < 0 || in->spatial_rank > 2) return -1;
  or_desc d; norm_desc(in, &d);
  if (d.cin < 1 || d.cout < 1 || d.groups < 1) return -1;
  if (d.cin % d.groups || d.cout % d.groups) return -1;
  for (int a = 0; a < 3; ++a)
    if (d.kernel[a] < 1 || d.stride[a] < 1 || d.dilation[a] < 1 || d.padding[a] < 0) return -1;
  for (int a = 0; a < 2; ++a) if (d.in_spatial[a] < 1) return -1;
  if (d.kernel[0] > 64) return -1;                 /* fixed-size window arrays below */
  /* S:51 "p <= f - 1 is enforced at construction" */
  if (d.padding[0] > or_receptive_field(&d) - 1) return -1;
  int out[2];
  or_out_spatial(&d, out);
  if (out[0] < 1 || out[1] < 1) return -1;
  return 0;
}

int or_receptive_field(const or_desc* d) {
  /* A5: the temporal extent of a dilated kernel, f = dil_t (kt - 1) + 1. */
  return d->dilation[0] * (d->kernel[0] - 1) + 1;
}

int or_delay(const or_desc* d) {
  /* Principle 4: d = f - p - 1. */
  return or_receptive_field(d) - d->padding[0] - 1;
}

int or_out_spatial(const or_desc* in, int out[2]) {
  or_desc d; norm_desc(in, &d);
  for (int a = 1; a <= 2; ++a) {
    long num = (long)d.in_spatial[a - 1] + 2L * d.padding[a] - (long)d.dilation[a] * (d.kernel[a] - 1) - 1;
    out[a - 1] = (num < 0) ? 0 : (int)(num / d.stride[a] + 1);
  }
  return 0;
}

int or_out_len(const or_desc* d, int T) {
  /* T' = floor((T + 2p - f)/s) + 1 */
  long num = (long)T + 2L * d->padding[0] - or_receptive_field(d);
  return (int)(floor_div(num, d->stride[0]) + 1);
}

int or_ring_slots(const or_desc* d) {
  int f = or_receptive_field(d);
  return (int)ceil_div(f - 1, d->stride[0]);
}

/* ---------------------------------------------------------------- O1 */

double or_column_at(const or_desc* in, const double* W, const double* bias,
                    const or_frame* Z, int o, int ho, int wo) {
  /* y[o,h',w'] = b[o] + sum_k sum_{c'<Cin/g} sum_{u,v}
   *     W[o,c',k,u,v] * Z_k[g(o) Cin/g + c', h' s_h + u dil_h - p_h, w' s_w + v dil_w - p_w]
   * (cross-correlation; out-of-range pixels read 0; g(o) = o / (Cout/g)). */
  or_desc d; norm_desc(in, &d);
  const int kt = d.kernel[0], kh = d.kernel[1], kw = d.kernel[2];
  const int cig = d.cin / d.groups, cog = d.cout / d.groups, g = o / cog;
  const int H = d.in_spatial[0], Wd = d.in_spatial[1];
  double acc = bias ? bias[o] : 0.0;
  for (int k = 0; k < kt; ++k) {
    if (!Z[k].p) continue;                         /* zero frame */
    for (int c = 0; c < cig; ++c) {
      const int ci = g * cig + c;
      for (int u = 0; u < kh; ++u) {
        const int hi = ho * d.stride[1] + u * d.dilation[1] - d.padding[1];
        if (hi < 0 || hi >= H) continue;
        for (int v = 0; v < kw; ++v) {
          const int wi = wo * d.stride[2] + v * d.dilation[2] - d.padding[2];
          if (wi < 0 || wi >= Wd) continue;
          const double w = W[((((long)o * cig + c) * kt + k) * kh + u) * kw + v];
          const double z = Z[k].p[(long)ci * Z[k].sc + (long)hi * Z[k].sh + (long)wi * Z[k].sw];
          acc += w * z;
        }
      }
    }
  }
  return acc;
}

void or_column(const or_desc* d, const double* W, const double* bias,
               const or_frame* Z, double* y, long y_sc) {
  int out[2];
  or_out_spatial(d, out);
  for (int o = 0; o < d->cout; ++o)
    for (int ho = 0; ho < out[0]; ++ho)
      for (int wo = 0; wo < out[1]; ++wo)
        y[(long)o * y_sc + (long)ho * out[1] + wo] = or_column_at(d, W, bias, Z, o, ho, wo);
}

/* ---------------------------------------------------------------- O2 */

int or_forward(const or_desc* in, const double* W, const double* bias,
               int B, const double* x, int T, double* y) {
  or_desc d; norm_desc(in, &d);
  const int Tp = or_out_len(&d, T);
  if (Tp < 1) return -1;                           /* S:63-65 insufficient length */
  const int kt = d.kernel[0], s = d.stride[0], dil = d.dilation[0], p = d.padding[0];
  const long HW = (long)d.in_spatial[0] * d.in_spatial[1];
  int out[2]; or_out_spatial(&d, out);
  const long HWo = (long)out[0] * out[1];
  or_frame* Zall = (or_frame*)malloc(sizeof(or_frame) * (size_t)kt * B * Tp);
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < Tp; ++i) {
      or_frame* Z = Zall + ((long)b * Tp + i) * kt;
      for (int k = 0; k < kt; ++k) {
        /* padded index q = i s + k dil; real frame t = q - p (zero outside [0,T)) */
        const long t = (long)i * s + (long)k * dil - p;
        if (t < 0 || t >= T) { Z[k].p = NULL; continue; }
        Z[k].p = x + ((long)b * d.cin * T + t) * HW;
        Z[k].sc = (long)T * HW; Z[k].sh = d.in_spatial[1]; Z[k].sw = 1;
      }
      or_column(&d, W, bias, Z, y + ((long)b * d.cout * Tp + i) * HWo, (long)Tp * HWo);
    }
  free(Zall);
  return Tp;
}

/* ---------------------------------------------------------------- O3 / O4 / O5 */

struct or_step {
  or_desc d;
  double* W; double* bias;
  int B, f, p, s, dil, kt, delay, R;
  long frame_elems;     /* B * Cin * S1 * S2 */
  long out_elems;       /* B * Cout * S1' * S2' */
  double* hist;         /* f-1 frames; hist[j] = padded frame m-(f-1)+j, m = n + p */
  long n;               /* stateful steps since clean_state() */
};

or_step* or_step_new(const or_desc* in, const double* W, const double* bias, int B) {
  if (or_validate(in) != 0 || B < 1) return NULL;
  or_step* sm = (or_step*)calloc(1, sizeof(or_step));
  norm_desc(in, &sm->d);
  const or_desc* d = &sm->d;
  sm->B = B;
  sm->f = or_receptive_field(d);
  sm->p = d->padding[0]; sm->s = d->stride[0]; sm->dil = d->dilation[0]; sm->kt = d->kernel[0];
  sm->delay = or_delay(d);
  sm->R = or_ring_slots(d);
  const long wn = (long)d->cout * (d->cin / d->groups) * d->kernel[0] * d->kernel[1] * d->kernel[2];
  sm->W = (double*)malloc(sizeof(double) * wn);
  memcpy(sm->W, W, sizeof(double) * wn);
  if (bias) {
    sm->bias = (double*)malloc(sizeof(double) * d->cout);
    memcpy(sm->bias, bias, sizeof(double) * d->cout);
  }
  int out[2]; or_out_spatial(d, out);
  sm->frame_elems = (long)B * d->cin * d->in_spatial[0] * d->in_spatial[1];
  sm->out_elems = (long)B * d->cout * out[0] * out[1];
  sm->hist = (double*)calloc((size_t)(sm->f > 1 ? sm->f - 1 : 1) * sm->frame_elems, sizeof(double));
  sm->n = 0;
  return sm;
}

void or_step_free(or_step* sm) {
  if (!sm) return;
  free(sm->W); free(sm->bias); free(sm->hist); free(sm);
}

void or_step_clean(or_step* sm) {
  /* P:116 clean_state(); P:213 / A8: the start padding "saturates" the state
   * with zero frames, and the clock restarts at n = 0. */
  memset(sm->hist, 0, sizeof(double) * (size_t)(sm->f > 1 ? sm->f - 1 : 1) * sm->frame_elems);
  sm->n = 0;
}

long or_step_count(const or_step* sm) { return sm->n; }

int or_step_head(const or_step* sm) {
  if (sm->R == 0) return 0;
  return (int)floor_mod(ceil_div(sm->n - sm->delay, sm->s), sm->R);
}

/* stream-local view of history frame j (0 <= j < f-1) */
static or_frame hist_frame(const or_step* sm, int j, int b) {
  or_frame z;
  const long HW = (long)sm->d.in_spatial[0] * sm->d.in_spatial[1];
  z.p = sm->hist + (long)j * sm->frame_elems + (long)b * sm->d.cin * HW;
  z.sc = HW; z.sh = sm->d.in_spatial[1]; z.sw = 1;
  return z;
}

int or_step_forward(or_step* sm, const double* x, int update_state, double* y) {
  const or_desc* d = &sm->d;
  const long HW = (long)d->in_spatial[0] * d->in_spatial[1];
  int out[2]; or_out_spatial(d, out);
  const long HWo = (long)out[0] * out[1];
  /* S:73 / S:125: Ready iff n >= d and (n - d) mod s == 0. */
  const int ready = (sm->n >= sm->delay) && (floor_mod(sm->n - sm->delay, sm->s) == 0);
  if (ready) {
    /* The output is batch column i = (n-d)/s; its window is the padded frames
     * i s + k dil = m-(f-1) + k dil, k = 0..kt-1 (m = n + p is the padded index of
     * x).  Window position k dil < f-1 is history frame k dil; k = kt-1 is x. */
#pragma omp parallel for schedule(static)
    for (int b = 0; b < sm->B; ++b) {
      or_frame Z[64];
      for (int k = 0; k < sm->kt; ++k) {
        const int j = k * sm->dil;
        if (j < sm->f - 1) {
          Z[k] = hist_frame(sm, j, b);
        } else if (x) {
          Z[k].p = x + (long)b * d->cin * HW; Z[k].sc = HW; Z[k].sh = d->in_spatial[1]; Z[k].sw = 1;
        } else {
          Z[k].p = NULL;
        }
      }
      or_column(d, sm->W, sm->bias, Z, y + (long)b * d->cout * HWo, HWo);
    }
  }
  if (update_state) {
    /* Push x (or a zero frame) into the history of the last f-1 padded frames. */
    if (sm->f > 1) {
      memmove(sm->hist, sm->hist + sm->frame_elems, sizeof(double) * (size_t)(sm->f - 2) * sm->frame_elems);
      double* last = sm->hist + (long)(sm->f - 2) * sm->frame_elems;
      if (x) memcpy(last, x, sizeof(double) * sm->frame_elems);
      else memset(last, 0, sizeof(double) * sm->frame_elems);
    }
    sm->n += 1;
  }
  return ready;
}

int or_step_forward_steps(or_step* sm, const double* x, int T, int pad_end,
                          int update_state, uint8_t* ready_mask, double* y) {
  /* P:94 "identical to applying forward_step the number of times corresponding
   * to the temporal size of the input"; P:215 pad_end feeds p zero steps.
   * With update_state = 0 the whole fold runs on a copy of the state. */
  const or_desc* d = &sm->d;
  const long HW = (long)d->in_spatial[0] * d->in_spatial[1];
  int out[2]; or_out_spatial(d, out);
  const long HWo = (long)out[0] * out[1];
  const int total = T + (pad_end ? sm->p : 0);
  or_step* run = sm;
  if (!update_state) {
    run = or_step_new(d, sm->W, sm->bias, sm->B);
    memcpy(run->hist, sm->hist, sizeof(double) * (size_t)(sm->f > 1 ? sm->f - 1 : 1) * sm->frame_elems);
    run->n = sm->n;
  }
  double* frame = (double*)malloc(sizeof(double) * sm->frame_elems);
  double* col = (double*)malloc(sizeof(double) * sm->out_elems);
  int n_ready = 0;
  for (int t = 0; t < total; ++t) {
    const double* xt = NULL;
    if (t < T) {
      for (int b = 0; b < sm->B; ++b)
        for (int c = 0; c < d->cin; ++c)
          memcpy(frame + ((long)b * d->cin + c) * HW, x + (((long)b * d->cin + c) * T + t) * HW,
                 sizeof(double) * HW);
      xt = frame;
    }
    const int r = or_step_forward(run, xt, 1, col);
    ready_mask[t] = (uint8_t)r;
    if (r) {
      /* compact in time (A1): y is (B, Cout, n_ready_total, S1', S2')
       * with n_ready_total = the number of Ready ticks; the caller sizes it. */
      for (int b = 0; b < sm->B; ++b)
        for (int o = 0; o < d->cout; ++o)
          memcpy(y + (((long)b * d->cout + o) * total + n_ready) * HWo,
                 col + ((long)b * d->cout + o) * HWo, sizeof(double) * HWo);
      n_ready++;
    }
  }
  free(frame); free(col);
  if (run != sm) or_step_free(run);
  return n_ready;   /* NOTE: y's time axis is allocated with `total` entries; first n_ready used */
}

void or_step_state(const or_step* sm, double* state) {
  const or_desc* d = &sm->d;
  int out[2]; or_out_spatial(d, out);
  const long HWo = (long)out[0] * out[1];
  const long m_next = sm->n + sm->p;                        /* next padded frame to consume */
  const long i_next = ceil_div(sm->n - sm->delay, sm->s);   /* next output to complete */
  for (int j = 0; j < sm->R; ++j) {
    const long i = i_next + j;
#pragma omp parallel for schedule(static)
    for (int b = 0; b < sm->B; ++b) {
      double* dst = state + (((long)j * sm->B + b) * d->cout) * HWo;
      if (i < 0) { memset(dst, 0, sizeof(double) * d->cout * HWo); continue; }
      or_frame Z[64];
      for (int k = 0; k < sm->kt; ++k) {
        const long q = i * sm->s + (long)k * sm->dil;     /* padded frame feeding slice k */
        if (q >= m_next) { Z[k].p = NULL; continue; }     /* not consumed yet */
        const long jj = q - (m_next - (sm->f - 1));       /* its history position */
        Z[k] = hist_frame(sm, (int)jj, b);
      }
      or_column(d, sm->W, NULL, Z, dst, HWo);             /* bias excluded (A9) */
    }
  }
}

/* The raw history itself (SPEC's state): the last f-1 padded
 * frames, oldest first, hist[j] = padded frame m_next-(f-1)+j, frames before
 * the start padding and the start padding itself being zero.  Read-only
 * accessor (no arithmetic): the CUDA path's raw-input-ring layout (SURVEY
 * §8f f1) exposes exactly this through co_state_get. */
void or_step_history(const or_step* sm, double* out) {
  memcpy(out, sm->hist, sizeof(double) * (size_t)(sm->f - 1) * sm->frame_elems);
}

/* ---------------------------------------------------------------- O7 */

int or_bruteforce_tick(const or_desc* in, const double* W, const double* bias,
                       int B, const double* hist, int n_plus_1, double* y) {
  or_desc d; norm_desc(in, &d);
  const long n = n_plus_1 - 1;
  const int delay = or_delay(&d), s = d.stride[0], p = d.padding[0];
  if (!(n >= delay && floor_mod(n - delay, s) == 0)) return 0;
  const long HW = (long)d.in_spatial[0] * d.in_spatial[1];
  const int L = p + n_plus_1;                              /* [p zeros | x_0..x_n] */
  double* z = (double*)calloc((size_t)B * d.cin * L * HW, sizeof(double));
  for (int b = 0; b < B; ++b)
    for (int c = 0; c < d.cin; ++c)
      memcpy(z + (((long)b * d.cin + c) * L + p) * HW, hist + (((long)b * d.cin + c) * n_plus_1) * HW,
             sizeof(double) * n_plus_1 * HW);
  or_desc d0 = d; d0.padding[0] = 0;
  const int Tp = or_out_len(&d0, L);
  int out[2]; or_out_spatial(&d, out);
  const long HWo = (long)out[0] * out[1];
  double* yy = (double*)malloc(sizeof(double) * (size_t)B * d.cout * Tp * HWo);
  or_forward(&d0, W, bias, B, z, L, yy);
  const long i = (n - delay) / s;                          /* == Tp - 1 */
  for (int b = 0; b < B; ++b)
    for (int o = 0; o < d.cout; ++o)
      memcpy(y + ((long)b * d.cout + o) * HWo, yy + (((long)b * d.cout + o) * Tp + i) * HWo,
             sizeof(double) * HWo);
  free(z); free(yy);
  return 1;
}

/* ---------------------------------------------------------------- O6 */

struct or_stack {
  int L, B;
  or_step** layers;
  int* relu; int* rnd;
  double** buf;
};

or_stack* or_stack_new(int n_layers, const or_desc* descs, const double* const* Ws,
                       const double* const* biases, const int* relu, const int* round_bf16, int B) {
  or_stack* st = (or_stack*)calloc(1, sizeof(or_stack));
  st->L = n_layers; st->B = B;
  st->layers = (or_step**)calloc(n_layers, sizeof(or_step*));
  st->relu = (int*)calloc(n_layers, sizeof(int));
  st->rnd = (int*)calloc(n_layers, sizeof(int));
  st->buf = (double**)calloc(n_layers, sizeof(double*));
  for (int l = 0; l < n_layers; ++l) {
    st->layers[l] = or_step_new(&descs[l], Ws[l], biases ? biases[l] : NULL, B);
    if (!st->layers[l]) { or_stack_free(st); return NULL; }
    st->relu[l] = relu ? relu[l] : 0;
    st->rnd[l] = round_bf16 ? round_bf16[l] : 0;
    st->buf[l] = (double*)malloc(sizeof(double) * st->layers[l]->out_elems);
  }
  return st;
}

void or_stack_free(or_stack* st) {
  if (!st) return;
  for (int l = 0; l < st->L; ++l) { or_step_free(st->layers[l]); free(st->buf ? st->buf[l] : NULL); }
  free(st->layers); free(st->relu); free(st->rnd); free(st->buf); free(st);
}

void or_stack_clean(or_stack* st) {
  for (int l = 0; l < st->L; ++l) or_step_clean(st->layers[l]);
}

int or_stack_forward(or_stack* st, const double* x, int update_state, double* y) {
  /* Sequential: thread the step value through the layers; an
   * Empty output ends the tick and the downstream layers are not advanced
   * (A7). */
  const double* cur = x;
  for (int l = 0; l < st->L; ++l) {
    if (!or_step_forward(st->layers[l], cur, update_state, st->buf[l])) return 0;
    const long ne = st->layers[l]->out_elems;
    double* v = st->buf[l];
    for (long e = 0; e < ne; ++e) {
      double t = v[e];
      if (st->relu[l] && t < 0.0) t = 0.0;   /* P:437 nn.ReLU between layers */
      if (st->rnd[l]) t = or_bf16_round(t);  /* declared bf16 activation (A16) */
      v[e] = t;
    }
    cur = v;
  }
  memcpy(y, cur, sizeof(double) * st->layers[st->L - 1]->out_elems);
  return 1;
}

/* ---------------------------------------------------------------- timing */

void or_accumulate(int n, const int* f, const int* p, const int* s,
                   int* s_acc, int* p_acc, int* f_acc, int* d_acc) {
  /* P:233-234, P:251-252, P:256, P:260-261 in the reading of the worked example
   * P:268-277 (A3): p_acc = {2, 2 + 2*0}, f_acc = {3, 3 + (3-1)*2}. */
  for (int i = 0; i < n; ++i) {
    if (i == 0) {
      s_acc[0] = s[0]; p_acc[0] = p[0]; f_acc[0] = f[0];
    } else {
      s_acc[i] = s[i] * s_acc[i - 1];
      p_acc[i] = p_acc[i - 1] + p[i] * s_acc[i - 1];
      f_acc[i] = f_acc[i - 1] + (f[i] - 1) * s_acc[i - 1];
    }
    d_acc[i] = f_acc[i] - p_acc[i] - 1;
  }
}

int or_schedule_ready(int d_nn, int s_nn, long t) {
  return (t >= d_nn) && (floor_mod(t - d_nn, s_nn) == 0);
}

/* ---------------------------------------------------------------- bf16 */

double or_bf16_round(double x) {
  /* bfloat16: 1 sign, 8 exponent, 7 stored mantissa bits -> 8 significant bits,
   * normal range down to 2^-126, subnormal spacing 2^-133.  Round to nearest,
   * ties to even (nearbyint under the default FE_TONEAREST mode). */
  if (x == 0.0 || !isfinite(x)) return x;
  int e;
  const double m = frexp(x, &e);                 /* x = m 2^e, 0.5 <= |m| < 1 */
  double r;
  if (e - 8 < -133) r = ldexp(nearbyint(ldexp(x, 133)), -133);   /* subnormal */
  else r = ldexp(nearbyint(ldexp(m, 8)), e - 8);
  if (fabs(r) > 3.3895313892515355e38) r = copysign(INFINITY, x); /* > max bf16 */
  return r;
}

void or_bf16_round_array(double* x, long n) {
  for (long i = 0; i < n; ++i) x[i] = or_bf16_round(x[i]);
}

/* ---------------------------------------------------------------- cost */

double or_flops_step(const or_desc* in) {
  or_desc d; norm_desc(in, &d);
  int out[2]; or_out_spatial(&d, out);
  return 2.0 * d.cout * (d.cin / d.groups) * d.kernel[0] * d.kernel[1] * d.kernel[2] * out[0] * out[1];
}
