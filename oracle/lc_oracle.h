/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * Plain-C restatement of the reference serve path (latecache, /root/reference/proj):
 *   lco_forward   <- forward()            src/network.cpp:104-164
 *   lco_softmax   <- softmax()            src/losses.cpp:35-46
 *   lco_sigmoid   <- sigmoid()            src/losses.cpp:26-33
 *   lco_argmax    <- argmax()             include/latecache/tensor.hpp:57-63
 *   lco_lookup    <- lookup()             src/cache.cpp:259-265
 *   lco_serve_mlp <- serve_one()          src/serving.cpp:97-124 (base = make_base_model net)
 * Pinned bit-exactly against the compiled reference (oracle/_ref) and the
 * golden fixtures in tests/golden/ (tests/test_oracle.py).
 *
 * CNN tier (no reference counterpart — "parity unpinned by reference" for the
 * base layers; cross-checked against torch fp64 in tests): NCHW fp64 conv2d,
 * per-channel affine (folded batch-norm), residual add, ReLU, max-pool and
 * global average pool, driven by an op list (lco_cnn_forward).
 */
#ifndef LC_ORACLE_H
#define LC_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { LCO_FC = 0, LCO_RELU = 1, LCO_POOL = 2, LCO_CONV1D = 3, LCO_SOFTMAX = 4 };

typedef struct {
  int kind;
  int in_dim, out_dim;
  int pool_window; /* average pool */
  int kernel, stride; /* conv1d */
  const double* w; /* fc: [out, in] row-major; conv1d: [kernel] */
  const double* b; /* fc: [out]; conv1d: [1] */
} lco_layer;

/* Runs the layer chain. `acts` (nullable) receives every activation,
 * input first, concatenated (sum of in_dim of layer 0 and out_dim of every
 * layer). Returns 0, or -1 on a dimension mismatch. */
int lco_forward(const lco_layer* layers, int n, const double* x, double* out, double* acts);
double lco_sigmoid(double x);
void lco_softmax(const double* x, int n, double* out);
int lco_argmax(const double* x, int n);

/* pr[classes] (nullable), logits[classes] (nullable). Returns hit (0/1). */
int lco_lookup(const lco_layer* pred, int np, const lco_layer* sel, int ns, double delta, const double* tap,
               double* prob, double* pr, double* logits);

typedef struct {
  int layer; /* 1-based tap index */
  const lco_layer* pred;
  int np;
  const lco_layer* sel;
  int ns;
  double delta;
} lco_cache;

/* serve_one over a make_base_model network: taps are the outputs of layers
 * tap_layer[i]; caches sorted by ascending layer; stops at the first hit.
 * probs[L] (nullable) receives the selector probability of every probed layer
 * (NaN for unprobed). Returns 0 or -1. */
int lco_serve_mlp(const lco_layer* base, int nb, const int* tap_layer, int blocks, const lco_cache* caches, int nc,
                  const double* x, int* exit_layer, int* served, int* base_pred, double* probs);

/* ------------------------------------------------------------ CNN tier */
enum { LCO_OP_CONV = 0, LCO_OP_MAXPOOL = 1, LCO_OP_GAP_FC = 2, LCO_OP_FC = 3 };

typedef struct {
  int op;
  int in_buf, out_buf, res_buf; /* buffer slots; res_buf = -1 for none */
  int C, H, W;                  /* input geometry (NCHW, per image) */
  int Cout, kh, kw, stride, pad;
  int relu;
  const double* w;     /* conv: [Cout][C][kh][kw]; fc: [Cout][C] */
  const double* scale; /* per Cout (nullable = 1) */
  const double* shift; /* per Cout (nullable = 0); fc bias */
  int tap;             /* >= 0: output of this op is tap #tap */
} lco_cnn_op;

/* Forward one image. bufs: nbufs scratch buffers of buf_len doubles each.
 * taps[t] receives the NCHW-flattened tap t (nullable entries skipped).
 * logits: final FC output. */
int lco_cnn_forward(const lco_cnn_op* ops, int nops, double** bufs, const double* x, double** taps, double* logits);

/* Batch forward on `threads` pthreads (independent images).
 * x: [B][in]; taps_out[t]: [B][tap_dim[t]] (nullable); logits: [B][classes]. */
int lco_cnn_forward_batch(const lco_cnn_op* ops, int nops, int nbufs, size_t buf_len, const double* x, size_t in_len,
                          int B, int ntaps, double** taps_out, const size_t* tap_dims, double* logits, int classes,
                          int threads);

/* ------------------------------------------------------------ RNG (rng.hpp:15-98)
 * splitmix64 / xoshiro256** / Box-Muller with a spare, mix_seed: the reference's
 * stream derivation. Used by oracle/cnn_models.py to rebuild the synthetic CNN
 * weights without the product library (the reference arm of bench.py). */
typedef struct {
  unsigned long long s[4];
  int has_spare;
  double spare;
} lco_rng;
unsigned long long lco_mix_seed(unsigned long long seed, unsigned long long tag);
void lco_rng_init(lco_rng* r, unsigned long long seed);
double lco_rng_uniform(lco_rng* r, double lo, double hi);
double lco_rng_normal(lco_rng* r);
/* out[i] = normal() * scale, i < n */
void lco_rng_normal_fill(lco_rng* r, double* out, size_t n, double scale);
/* out[i] = uniform(lo, hi), i < n */
void lco_rng_uniform_fill(lco_rng* r, double* out, size_t n, double lo, double hi);
/* per channel c: scale[c] = gain * uniform(0.8, 1.2); shift[c] = uniform(-0.1, 0.1) */
void lco_rng_bn_fill(lco_rng* r, int n, double gain, double* scale, double* shift);

#ifdef __cplusplus
}
#endif
#endif
