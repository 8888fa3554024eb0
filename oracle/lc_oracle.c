/* TEST INFRASTRUCTURE ONLY — CPU oracle. See lc_oracle.h for the citations.
 * Compiled with -ffp-contract=off so every multiply-add rounds like the
 * reference's scalar loops. */
#include "lc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* network.cpp:104-164 */
int lco_forward(const lco_layer* L, int n, const double* x, double* out, double* acts) {
  if (n <= 0) return -1;
  int maxd = L[0].in_dim;
  for (int i = 0; i < n; ++i) {
    if (i > 0 && L[i].in_dim != L[i - 1].out_dim) return -1;
    if (L[i].out_dim > maxd) maxd = L[i].out_dim;
  }
  double* a = (double*)malloc(sizeof(double) * (size_t)maxd);
  double* y = (double*)malloc(sizeof(double) * (size_t)maxd);
  memcpy(a, x, sizeof(double) * (size_t)L[0].in_dim);
  size_t aoff = 0;
  if (acts) {
    memcpy(acts, x, sizeof(double) * (size_t)L[0].in_dim);
    aoff = (size_t)L[0].in_dim;
  }
  for (int i = 0; i < n; ++i) {
    const lco_layer* s = &L[i];
    switch (s->kind) {
      case LCO_FC:
        for (int o = 0; o < s->out_dim; ++o) {
          double acc = s->b[o];
          const double* row = s->w + (size_t)o * (size_t)s->in_dim;
          for (int j = 0; j < s->in_dim; ++j) acc += row[j] * a[j];
          y[o] = acc;
        }
        break;
      case LCO_RELU:
        for (int j = 0; j < s->in_dim; ++j) y[j] = a[j] > 0.0 ? a[j] : 0.0;
        break;
      case LCO_POOL: {
        const double inv = 1.0 / s->pool_window;
        for (int o = 0; o < s->out_dim; ++o) {
          double acc = 0.0;
          for (int t = 0; t < s->pool_window; ++t) acc += a[o * s->pool_window + t];
          y[o] = acc * inv;
        }
        break;
      }
      case LCO_CONV1D: {
        const double b = s->b[0];
        for (int o = 0; o < s->out_dim; ++o) {
          double acc = b;
          for (int t = 0; t < s->kernel; ++t) acc += s->w[t] * a[o * s->stride + t];
          y[o] = acc;
        }
        break;
      }
      case LCO_SOFTMAX: {
        double m = a[0];
        for (int j = 1; j < s->in_dim; ++j) m = (m < a[j]) ? a[j] : m; /* std::max */
        double sum = 0.0;
        for (int j = 0; j < s->in_dim; ++j) {
          y[j] = exp(a[j] - m);
          sum += y[j];
        }
        for (int j = 0; j < s->in_dim; ++j) y[j] /= sum;
        break;
      }
      default:
        free(a);
        free(y);
        return -1;
    }
    double* t = a;
    a = y;
    y = t;
    if (acts) {
      memcpy(acts + aoff, a, sizeof(double) * (size_t)s->out_dim);
      aoff += (size_t)s->out_dim;
    }
  }
  memcpy(out, a, sizeof(double) * (size_t)L[n - 1].out_dim);
  free(a);
  free(y);
  return 0;
}

/* losses.cpp:26-33 */
double lco_sigmoid(double x) {
  if (x >= 0.0) {
    const double z = exp(-x);
    return 1.0 / (1.0 + z);
  }
  const double z = exp(x);
  return z / (1.0 + z);
}

/* losses.cpp:35-46 */
void lco_softmax(const double* x, int n, double* out) {
  double m = x[0];
  for (int i = 1; i < n; ++i) m = (m < x[i]) ? x[i] : m;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    out[i] = exp(x[i] - m);
    sum += out[i];
  }
  for (int i = 0; i < n; ++i) out[i] /= sum;
}

/* tensor.hpp:57-63: ties resolve to the smallest index */
int lco_argmax(const double* x, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (x[i] > x[best]) best = i;
  return best;
}

/* cache.cpp:259-265 */
int lco_lookup(const lco_layer* pred, int np, const lco_layer* sel, int ns, double delta, const double* tap,
               double* prob, double* pr, double* logits) {
  const int C = pred[np - 1].out_dim;
  double* lg = (double*)malloc(sizeof(double) * (size_t)C);
  double* p = (double*)malloc(sizeof(double) * (size_t)C);
  double z = 0.0;
  lco_forward(pred, np, tap, lg, NULL);
  lco_softmax(lg, C, p);
  lco_forward(sel, ns, p, &z, NULL);
  const double q = lco_sigmoid(z);
  if (prob) *prob = q;
  if (pr) memcpy(pr, p, sizeof(double) * (size_t)C);
  if (logits) memcpy(logits, lg, sizeof(double) * (size_t)C);
  free(lg);
  free(p);
  return q >= delta ? 1 : 0; /* inclusive threshold */
}

/* serving.cpp:97-124 */
int lco_serve_mlp(const lco_layer* base, int nb, const int* tap_layer, int blocks, const lco_cache* caches, int nc,
                  const double* x, int* exit_layer, int* served, int* base_pred, double* probs) {
  size_t total = (size_t)base[0].in_dim;
  for (int i = 0; i < nb; ++i) total += (size_t)base[i].out_dim;
  double* acts = (double*)malloc(sizeof(double) * total);
  const int C = base[nb - 1].out_dim;
  double* y = (double*)malloc(sizeof(double) * (size_t)C);
  if (lco_forward(base, nb, x, y, acts) != 0) {
    free(acts);
    free(y);
    return -1;
  }
  /* offsets of each layer's output inside acts */
  size_t* off = (size_t*)malloc(sizeof(size_t) * (size_t)(nb + 1));
  off[0] = 0;
  size_t cur = (size_t)base[0].in_dim;
  for (int i = 0; i < nb; ++i) {
    off[i + 1] = cur;
    cur += (size_t)base[i].out_dim;
  }
  *base_pred = lco_argmax(y, C);
  *served = *base_pred;
  *exit_layer = 0;
  if (probs)
    for (int l = 0; l < blocks; ++l) probs[l] = NAN;
  double* pr = (double*)malloc(sizeof(double) * (size_t)C);
  for (int k = 0; k < nc; ++k) {
    const int layer = caches[k].layer;
    const double* tap = acts + off[tap_layer[layer - 1] + 1];
    double q = 0.0;
    const int hit = lco_lookup(caches[k].pred, caches[k].np, caches[k].sel, caches[k].ns, caches[k].delta, tap, &q, pr,
                               NULL);
    if (probs) probs[layer - 1] = q;
    if (hit) {
      *served = lco_argmax(pr, caches[k].pred[caches[k].np - 1].out_dim);
      *exit_layer = layer;
      break;
    }
  }
  free(pr);
  free(off);
  free(acts);
  free(y);
  return 0;
}

/* ------------------------------------------------------------ CNN tier */
static void conv2d_nchw(const double* x, int C, int H, int W, const double* w, int Cout, int kh, int kw, int stride,
                        int pad, double* y, int Ho, int Wo) {
  for (int co = 0; co < Cout; ++co) {
    double* yo = y + (size_t)co * Ho * Wo;
    for (int i = 0; i < Ho * Wo; ++i) yo[i] = 0.0;
    for (int c = 0; c < C; ++c) {
      const double* xc = x + (size_t)c * H * W;
      const double* wc = w + ((size_t)co * C + c) * kh * kw;
      for (int r = 0; r < kh; ++r)
        for (int s = 0; s < kw; ++s) {
          const double wv = wc[r * kw + s];
          for (int oh = 0; oh < Ho; ++oh) {
            const int ih = oh * stride + r - pad;
            if (ih < 0 || ih >= H) continue;
            const double* xr = xc + (size_t)ih * W;
            double* yr = yo + (size_t)oh * Wo;
            for (int ow = 0; ow < Wo; ++ow) {
              const int iw = ow * stride + s - pad;
              if (iw < 0 || iw >= W) continue;
              yr[ow] += wv * xr[iw];
            }
          }
        }
    }
  }
}

int lco_cnn_forward(const lco_cnn_op* ops, int nops, double** bufs, const double* x, double** taps, double* logits) {
  const double* in0 = x;
  for (int k = 0; k < nops; ++k) {
    const lco_cnn_op* o = &ops[k];
    const double* in = o->in_buf < 0 ? in0 : bufs[o->in_buf];
    double* out = o->out_buf < 0 ? logits : bufs[o->out_buf];
    int outC = o->Cout, Ho = 1, Wo = 1;
    switch (o->op) {
      case LCO_OP_CONV: {
        Ho = (o->H + 2 * o->pad - o->kh) / o->stride + 1;
        Wo = (o->W + 2 * o->pad - o->kw) / o->stride + 1;
        conv2d_nchw(in, o->C, o->H, o->W, o->w, o->Cout, o->kh, o->kw, o->stride, o->pad, out, Ho, Wo);
        const size_t hw = (size_t)Ho * Wo;
        for (int co = 0; co < o->Cout; ++co) {
          const double sc = o->scale ? o->scale[co] : 1.0, sh = o->shift ? o->shift[co] : 0.0;
          double* yo = out + (size_t)co * hw;
          const double* ro = o->res_buf >= 0 ? bufs[o->res_buf] + (size_t)co * hw : NULL;
          for (size_t i = 0; i < hw; ++i) {
            double v = yo[i] * sc + sh;
            if (ro) v += ro[i];
            if (o->relu) v = v > 0.0 ? v : 0.0;
            yo[i] = v;
          }
        }
        break;
      }
      case LCO_OP_MAXPOOL: {
        outC = o->C;
        Ho = (o->H + 2 * o->pad - o->kh) / o->stride + 1;
        Wo = (o->W + 2 * o->pad - o->kw) / o->stride + 1;
        for (int c = 0; c < o->C; ++c)
          for (int oh = 0; oh < Ho; ++oh)
            for (int ow = 0; ow < Wo; ++ow) {
              double m = -INFINITY;
              for (int r = 0; r < o->kh; ++r)
                for (int s = 0; s < o->kw; ++s) {
                  const int ih = oh * o->stride + r - o->pad, iw = ow * o->stride + s - o->pad;
                  if (ih < 0 || ih >= o->H || iw < 0 || iw >= o->W) continue;
                  const double v = in[((size_t)c * o->H + ih) * o->W + iw];
                  if (v > m) m = v;
                }
              out[((size_t)c * Ho + oh) * Wo + ow] = m;
            }
        break;
      }
      case LCO_OP_GAP_FC: {
        /* global average pool over H*W then FC(C, Cout) with bias */
        const size_t hw = (size_t)o->H * o->W;
        double* g = (double*)malloc(sizeof(double) * (size_t)o->C);
        for (int c = 0; c < o->C; ++c) {
          double acc = 0.0;
          for (size_t i = 0; i < hw; ++i) acc += in[(size_t)c * hw + i];
          g[c] = acc * (1.0 / (double)hw);
        }
        for (int co = 0; co < o->Cout; ++co) {
          double acc = o->shift ? o->shift[co] : 0.0;
          for (int c = 0; c < o->C; ++c) acc += o->w[(size_t)co * o->C + c] * g[c];
          out[co] = acc;
        }
        free(g);
        break;
      }
      case LCO_OP_FC: {
        const size_t D = (size_t)o->C * o->H * o->W;
        for (int co = 0; co < o->Cout; ++co) {
          double acc = o->shift ? o->shift[co] : 0.0;
          for (size_t j = 0; j < D; ++j) acc += o->w[(size_t)co * D + j] * in[j];
          if (o->relu) acc = acc > 0.0 ? acc : 0.0;
          out[co] = acc;
        }
        break;
      }
      default:
        return -1;
    }
    if (o->tap >= 0 && taps && taps[o->tap]) {
      memcpy(taps[o->tap], out, sizeof(double) * (size_t)outC * Ho * Wo);
    }
  }
  return 0;
}

typedef struct {
  const lco_cnn_op* ops;
  int nops, nbufs, ntaps, classes, B, T, k;
  size_t buf_len, in_len;
  const double* x;
  double** taps_out;
  const size_t* tap_dims;
  double* logits;
  int err;
} lco_job;

static void* lco_worker(void* arg) {
  lco_job* j = (lco_job*)arg;
  double** bufs = (double**)malloc(sizeof(double*) * (size_t)j->nbufs);
  for (int i = 0; i < j->nbufs; ++i) bufs[i] = (double*)calloc(j->buf_len, sizeof(double));
  double** taps = (double**)malloc(sizeof(double*) * (size_t)(j->ntaps > 0 ? j->ntaps : 1));
  for (int b = j->k; b < j->B; b += j->T) {
    for (int t = 0; t < j->ntaps; ++t)
      taps[t] = (j->taps_out && j->taps_out[t]) ? j->taps_out[t] + (size_t)b * j->tap_dims[t] : NULL;
    if (lco_cnn_forward(j->ops, j->nops, bufs, j->x + (size_t)b * j->in_len, taps, j->logits + (size_t)b * j->classes))
      j->err = 1;
  }
  for (int i = 0; i < j->nbufs; ++i) free(bufs[i]);
  free(bufs);
  free(taps);
  return NULL;
}

/* Images are independent; `threads` pthreads take them round-robin. */
int lco_cnn_forward_batch(const lco_cnn_op* ops, int nops, int nbufs, size_t buf_len, const double* x, size_t in_len,
                          int B, int ntaps, double** taps_out, const size_t* tap_dims, double* logits, int classes,
                          int threads) {
  if (threads < 1) threads = 1;
  if (threads > B) threads = B;
  lco_job* jobs = (lco_job*)calloc((size_t)threads, sizeof(lco_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int k = 0; k < threads; ++k) {
    lco_job j = {ops, nops, nbufs, ntaps, classes, B, threads, k, buf_len, in_len, x, taps_out, tap_dims, logits, 0};
    jobs[k] = j;
  }
  for (int k = 1; k < threads; ++k) pthread_create(&th[k], NULL, lco_worker, &jobs[k]);
  lco_worker(&jobs[0]);
  int err = jobs[0].err;
  for (int k = 1; k < threads; ++k) {
    pthread_join(th[k], NULL);
    err |= jobs[k].err;
  }
  free(jobs);
  free(th);
  return err ? -1 : 0;
}

/* ------------------------------------------------------------ RNG
 * rng.hpp:15-98 restated: splitmix64 seeding, xoshiro256**, 53-bit doubles,
 * Box-Muller with a cached spare, mix_seed. */
static unsigned long long lco_splitmix64(unsigned long long* state) {
  unsigned long long z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

unsigned long long lco_mix_seed(unsigned long long seed, unsigned long long tag) {
  unsigned long long s = seed + 0x9e3779b97f4a7c15ULL * (tag + 0x632be59bd9b4e019ULL);
  const unsigned long long a = lco_splitmix64(&s);
  const unsigned long long b = lco_splitmix64(&s);
  return a ^ (b << 1);
}

void lco_rng_init(lco_rng* r, unsigned long long seed) {
  unsigned long long sm = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = lco_splitmix64(&sm);
  r->has_spare = 0;
  r->spare = 0.0;
}

static unsigned long long lco_rotl(unsigned long long x, int k) { return (x << k) | (x >> (64 - k)); }

static unsigned long long lco_next_u64(lco_rng* r) {
  unsigned long long* s = r->s;
  const unsigned long long result = lco_rotl(s[1] * 5, 7) * 9;
  const unsigned long long t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = lco_rotl(s[3], 45);
  return result;
}

static double lco_next_double(lco_rng* r) { return (double)(lco_next_u64(r) >> 11) * 0x1.0p-53; }

double lco_rng_uniform(lco_rng* r, double lo, double hi) { return lo + (hi - lo) * lco_next_double(r); }

double lco_rng_normal(lco_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = 1.0 - lco_next_double(r);
  const double u2 = lco_next_double(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(theta);
  r->has_spare = 1;
  return rad * cos(theta);
}

void lco_rng_normal_fill(lco_rng* r, double* out, size_t n, double scale) {
  for (size_t i = 0; i < n; ++i) out[i] = lco_rng_normal(r) * scale;
}

void lco_rng_uniform_fill(lco_rng* r, double* out, size_t n, double lo, double hi) {
  for (size_t i = 0; i < n; ++i) out[i] = lco_rng_uniform(r, lo, hi);
}

void lco_rng_bn_fill(lco_rng* r, int n, double gain, double* scale, double* shift) {
  for (int c = 0; c < n; ++c) {
    scale[c] = gain * lco_rng_uniform(r, 0.8, 1.2);
    shift[c] = lco_rng_uniform(r, -0.1, 0.1);
  }
}
