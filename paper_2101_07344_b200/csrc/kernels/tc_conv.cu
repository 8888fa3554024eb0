// tcgen05 / TMA / TMEM implicit-GEMM kernel. See tc_conv.cuh for the contract.
//
// Warp roles (320 threads, one CTA per SM, persistent over tiles):
//   warp 0      : TMA producer (lane 0) + TMEM allocator (whole warp)
//   warp 1      : MMA issuer (lane 0)
//   warps 2..9  : epilogue; warp w reads TMEM lane quadrant w % 4 and owns
//                 column half (w - 2) / 4 of the tile (two warps per quadrant)
// Pipelines: smem ring full/empty (TMA <-> MMA), TMEM double buffer
// tfull/tempty (MMA <-> epilogue), split-K tile counters (CTA <-> CTA).
#include <cfloat>

#include "gpu_sync.cuh"
#include "pdl.cuh"
#include "sm100_prims.cuh"
#include "tc_conv.cuh"

namespace lcb {

namespace {

constexpr int kBM = 128;
constexpr int kABytes = kBM * 128;  // 128 rows x 64 bf16

template <int BN, bool X3>
struct TcCfg {
  static constexpr int kPlanes = X3 ? 2 : 1;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStageBytes = kPlanes * (kABytes + kBBytes);
  static constexpr int kStagesRaw = (192 * 1024) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kEpiWarpBytes = kPlanes * 2048;  // per epilogue warp: 32 rows x 64 B per plane
  static constexpr int kEpiStage = 8 * kEpiWarpBytes;
  static constexpr int kShiftBytes = 2 * BN * 4;  // per-tile shift values, double-buffered with the accumulators
  static constexpr int kSmem = kStages * kStageBytes + kEpiStage + 1024 /*bars*/ + kShiftBytes + 1024 /*align*/;
  // bf16x3 accumulators are 2*BN columns wide: with p.stacked the hi*hi and
  // hi*lo products are ONE N = 2*BN MMA over the stage's contiguous
  // [B_hi; B_lo] rows into [cols 0, BN) and [BN, 2BN), lo*hi goes into the
  // low half, and the epilogue adds the halves (2 MMAs per K16 group instead of
  // 3: an MMA costs ~38 + 0.375*N cycles and re-reads its A fragment).
  static constexpr int kAccCols = X3 ? 2 * BN : BN;
  static constexpr uint32_t kTmemCols = 2 * kAccCols;
  static_assert(kStages >= 2, "pipeline needs at least two stages");
};

// Division by a launch-constant divisor through a multiply-high (dividends
// < 2^31): the persistent loops decode a tile per iteration in every role, and
// runtime integer divisions were a large share of the epilogue's instructions.
struct FastDiv {
  uint32_t d, m, s;
  __device__ __forceinline__ void init(int div) {
    d = static_cast<uint32_t>(div < 1 ? 1 : div);
    if (d == 1) {
      m = 0;
      s = 0;
    } else {
      const uint32_t l = 32 - __clz(d - 1);  // ceil(log2 d)
      const uint32_t pw = 31 + l;
      if (d <= (1u << 20)) {
        // ceil(2^pw / d) from one correctly rounded double division: exact
        // for d <= 2^20 (a non-integer quotient < 2^32 stays >= 1/d > ulp
        // away from the integers). The u64 division below is a ~100-
        // instruction software routine on the kernel's startup path.
        m = static_cast<uint32_t>(ceil(__ddiv_rn(__longlong_as_double(static_cast<long long>(1023 + pw) << 52),
                                                 static_cast<double>(d))));
      } else {
        m = static_cast<uint32_t>(((1ull << pw) + d - 1) / d);
      }
      s = pw - 32;
    }
  }
  __device__ __forceinline__ int div(int x) const {
    return d == 1 ? x : static_cast<int>(__umulhi(static_cast<uint32_t>(x), m) >> s);
  }
  __device__ __forceinline__ void divmod(int x, int& q, int& r) const {
    q = div(x);
    r = x - q * static_cast<int>(d);
  }
};

struct TileGeom {
  int count, n_groups, tiles_w, tiles_img, tiles_n, tiles_mn, ks, total, nk;
  FastDiv fks, ftn, fimg, ftw;
};

__device__ __forceinline__ TileGeom tile_geom(const TcConvParams& p, int BN) {
  TileGeom g;
  g.count = p.count ? *p.count : p.count_static;
  if (p.plain) {
    g.n_groups = 1;
    g.tiles_w = (g.count + kBM - 1) / kBM;
  } else {
    g.n_groups = (g.count + p.ipt - 1) / p.ipt;
    g.tiles_w = p.tiles_w;
  }
  g.tiles_img = p.tiles_h * g.tiles_w;
  g.tiles_n = p.Cout / BN;
  g.tiles_mn = g.n_groups * g.tiles_img * g.tiles_n;
  g.nk = p.ntaps * (p.C / 64) + p.nres;
  if (p.mode == 1) {
    g.ks = p.ksplit;
  } else if (p.ks_max > 1 && g.tiles_mn > 0) {
    // Fill the grid as the surviving-request count shrinks. Floor, so that
    // tiles_mn * ks <= gridDim.x: every CTA owns at most one unit of a split
    // tile and all units of a tile are co-resident (the reduction waits on them).
    int ks = static_cast<int>(gridDim.x) / g.tiles_mn;
    ks = ks > p.ks_max ? p.ks_max : ks;
    ks = ks > g.nk ? g.nk : ks;
    if (p.ks_min_steps > 0) {
      const int cap = g.nk / p.ks_min_steps;
      ks = ks > cap ? cap : ks;
    }
    g.ks = ks < 1 ? 1 : ks;
  } else {
    g.ks = 1;
  }
  g.total = g.tiles_mn * g.ks;
  g.fks.init(g.ks);
  g.ftn.init(g.tiles_n);
  g.fimg.init(g.tiles_img);
  g.ftw.init(g.tiles_w);
  return g;
}

struct Tile {
  int tn, ks, tile_mn, grp, th, tw, h0, w0, s_begin, s_end;
};

__device__ __forceinline__ Tile decode_tile(int t, const TcConvParams& p, const TileGeom& g) {
  Tile x;
  int tm, r;
  g.fks.divmod(t, x.tile_mn, x.ks);
  g.ftn.divmod(x.tile_mn, tm, x.tn);
  g.fimg.divmod(tm, x.grp, r);
  g.ftw.divmod(r, x.th, x.tw);
  x.h0 = x.th * p.hb;
  x.w0 = x.tw * p.wb;
  if (g.ks == 1) {
    x.s_begin = 0;
    x.s_end = g.nk;
  } else {  // nk * ks < 2^31
    x.s_begin = g.fks.div(g.nk * x.ks);
    x.s_end = g.fks.div(g.nk * (x.ks + 1));
  }
  return x;
}

__device__ __forceinline__ int image_of(const TcConvParams& p, int idx) { return p.surv ? p.surv[idx] : idx; }

constexpr int kEpiUnroll = 2;  // 32-column epilogue steps unrolled together (BN = 128: r50 l1 64->256 227 -> 200 us)
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreads = 64 + kEpiThreads;
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }


__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

// Trace slot (debug instrumentation): CTA < kTraceCtas, unit < kTraceUnits.
constexpr int kTraceCtas = 8, kTraceUnits = 32, kTraceFields = 32;
__device__ __forceinline__ void trace_put(const TcConvParams& p, int unit, int field) {
  if (p.trace && blockIdx.x < kTraceCtas && unit < kTraceUnits)
    p.trace[(blockIdx.x * kTraceUnits + unit) * kTraceFields + field] = clk();
}

// Per-K-step wait/issue cycle counters (trace fields 12-14): compiled only
// with -DLCB_TC_TRACE (tests/cuda/tc_selftest), since the MMA warp is
// issue-bound and the extra instructions cost ~3 % in the library build.
#ifdef LCB_TC_TRACE
#define TC_TRACE(...) __VA_ARGS__
#else
#define TC_TRACE(...)
#endif
__device__ __forceinline__ void trace_val(const TcConvParams& p, int unit, int field, unsigned long long v) {
  if (p.trace && blockIdx.x < kTraceCtas && unit < kTraceUnits) p.trace[(blockIdx.x * kTraceUnits + unit) * kTraceFields + field] = v;
}

// Tile-invariant part of a tile row's output coordinates: image slot j and
// pixel offset (dh, dw) inside the ipt x hb x wb box (computed once per thread).
struct RowGeom {
  int j, dh, dw;
  FastDiv fpw;  // halo: padded row pitch
};
__device__ __forceinline__ RowGeom row_geom(const TcConvParams& p, int row) {
  RowGeom rg;
  rg.fpw.init(p.halo ? p.halo_pw : 1);
  if (p.plain || p.halo) {
    rg.j = rg.dh = rg.dw = 0;
  } else {
    const int rows_per_img = p.hb * p.wb;
    rg.j = row / rows_per_img;
    const int pix = row % rows_per_img;
    rg.dh = pix / p.wb;
    rg.dw = pix % p.wb;
  }
  return rg;
}

// Output element offset of tile row `row` (NHWC (n, h, w, 0) or plain row start).
// img: the row's image id (surviving-request slot resolved), img_ok: the
// tile's image slot exists (the row itself may still lie outside the image).
__device__ __forceinline__ bool out_row(const TcConvParams& p, const TileGeom& g, const Tile& x, int row,
                                        const RowGeom& rg, size_t& obase, int& img, bool& img_ok) {
  if (p.plain) {
    const int grow = x.w0 + row;
    obase = static_cast<size_t>(grow) * (p.out_ld > 0 ? p.out_ld : p.Cout);
    img = grow;
    img_ok = grow < g.count;
    return img_ok;
  }
  int idx, h, w;
  if (p.halo) {
    // anchors on the padded row pitch: m = oh * Pw + ow (ow >= Wo are discarded)
    const int m = x.h0 * kBM + row;
    rg.fpw.divmod(m, h, w);
    idx = x.grp;
  } else {
    h = x.h0 + rg.dh;
    w = x.w0 + rg.dw;
    idx = x.grp * p.ipt + rg.j;
  }
  img_ok = idx < g.count;
  const bool valid = img_ok && (h < p.Ho) && (w < p.Wo);
  const int n = img_ok ? (p.surv ? p.surv[idx] : idx) : 0;
  img = n;
  obase = ((static_cast<size_t>(n) * p.Ho + h) * p.Wo + w) * p.Cout;
  return valid;
}

// scale/shift, residual (prefetched 16-byte chunks), ReLU, hi/lo split and
// NHWC store of 16 channels.
// sh: the 16 shift values of these columns (shared-memory copy or global), nullable.
__device__ __forceinline__ void epilogue_math(const TcConvParams& p, float (&v)[16], int co, const float* sh,
                                              const uint4* rh, const uint4* rl) {
  if (p.scale) {
    const float4* sc = reinterpret_cast<const float4*>(p.scale + co);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 s4 = __ldg(sc + q);
      v[4 * q] *= s4.x;
      v[4 * q + 1] *= s4.y;
      v[4 * q + 2] *= s4.z;
      v[4 * q + 3] *= s4.w;
    }
  }
  if (sh) {
    const float4* sh4 = reinterpret_cast<const float4*>(sh);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 s4 = sh4[q];
      v[4 * q] += s4.x;
      v[4 * q + 1] += s4.y;
      v[4 * q + 2] += s4.z;
      v[4 * q + 3] += s4.w;
    }
  }
  if (rh) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&rh[q]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(b2[e]);
        v[8 * q + 2 * e] += f.x;
        v[8 * q + 2 * e + 1] += f.y;
      }
    }
    if (rl) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&rl[q]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(b2[e]);
          v[8 * q + 2 * e] += f.x;
          v[8 * q + 2 * e + 1] += f.y;
        }
      }
    }
  }
  if (p.relu) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = v[i] > 0.0f ? v[i] : 0.0f;
  }
}

__device__ __forceinline__ void split16(const float (&v)[16], uint4 (&hi)[2], uint4 (&lo)[2]) {
  __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(hi);
  __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(lo);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
    h2[e] = hh;
    const float2 hf = __bfloat1622float2(hh);
    l2[e] = __floats2bfloat162_rn(v[2 * e] - hf.x, v[2 * e + 1] - hf.y);
  }
}

__device__ __forceinline__ void epilogue_store(const TcConvParams& p, float (&v)[16], size_t off, int co,
                                               const uint4* rh, const uint4* rl) {
  epilogue_math(p, v, co, p.shift ? p.shift + co : nullptr, rh, rl);
  uint4 hi[2], lo[2];
  __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(hi);
  __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(lo);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
    h2[e] = hh;
    const float2 hf = __bfloat1622float2(hh);
    l2[e] = __floats2bfloat162_rn(v[2 * e] - hf.x, v[2 * e + 1] - hf.y);
  }
  uint4* oh = reinterpret_cast<uint4*>(p.out_hi + off);
  oh[0] = hi[0];
  oh[1] = hi[1];
  if (p.out_lo) {
    uint4* ol = reinterpret_cast<uint4*>(p.out_lo + off);
    ol[0] = lo[0];
    ol[1] = lo[1];
  }
}


// Fused global-average-pool partials of the tap this conv produces (the
// learned cache's Pool(C) = GAP predictor input, cache.cpp:104-140 with
// window H*W): the 32 lanes of a warp hold 32 consecutive tile rows (pixels)
// of one 16-channel chunk. A segmented reduce-scatter over the lane bits
// inside an image's run of rows (segments of min(rows_per_img, 32) rows)
// halves the live values at each xor step (16 -> 8 -> 4 -> 2 -> 1 values,
// 15-16 shuffles instead of 80, fixed order), leaving each lane with the
// segment sum of channel(s) selected by its lane bits; those lanes write the
// sums to gap_out[n][segment][Cout]. Every segment slot of every present
// image is written each launch (rows outside the image contribute 0), so the
// head sums all gap_segs slots.
// One halving step of the segmented reduce-scatter: lanes whose bit `o` is 0
// keep the lower kN/2 live values (adding the partner's), the others the upper.
template <int kN>
__device__ __forceinline__ void rs_step(float (&v)[16], int o, int lane) {
  const bool up = (lane & o) != 0;
#pragma unroll
  for (int e = 0; e < kN / 2; ++e) {
    const float send = up ? v[e] : v[e + kN / 2];
    const float keep = up ? v[e + kN / 2] : v[e];
    v[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
  }
}

// Segment size seg = min(rows_per_img, 32) in {8, 16, 32}: halvings over the
// lane bits seg/2, seg/4, seg/8 (and seg/16 when seg >= 16), plus a plain
// add over bit 0 for seg == 32. Value e of a lane is then channel chbase + e
// (2 live values for seg == 8, else 1).
// img / img_ok: this lane's image (every row of a segment lies in one image).
__device__ __forceinline__ void gap_segment(const TcConvParams& p, const Tile& x, int row, int lane, float (&v)[16],
                                            int co, int img, bool img_ok) {
  const int rpi = p.halo ? kBM : p.hb * p.wb;  // power of two >= 8
  const int seg = rpi < 32 ? rpi : 32;
  rs_step<16>(v, seg >> 1, lane);
  rs_step<8>(v, seg >> 2, lane);
  rs_step<4>(v, seg >> 3, lane);
  int chbase = ((lane & (seg >> 1)) ? 8 : 0) + ((lane & (seg >> 2)) ? 4 : 0) + ((lane & (seg >> 3)) ? 2 : 0);
  bool writer = true;
  if (seg >= 16) {
    rs_step<2>(v, seg >> 4, lane);
    chbase += (lane & (seg >> 4)) ? 1 : 0;
  }
  if (seg == 32) {
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    writer = (lane & 1) == 0;
  }
  const int seg_first = row & ~(seg - 1);  // first row of this lane's segment
  if (writer && img_ok) {
    const int pix = seg_first & (rpi - 1);
    const int per_tile = rpi > 32 ? rpi >> 5 : 1;
    const int tile_r = x.th * p.tiles_w + x.tw;
    const int sg = tile_r * per_tile + (pix >> 5);
    float* dst = p.gap_out + (static_cast<size_t>(img) * p.gap_segs + sg) * p.Cout + co + chbase;
    dst[0] = v[0];
    if (seg == 8) dst[1] = v[1];
  }
}

// ------------------------------------------------------------ fused lookup
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// First-hit exit + stable compaction over the layer's n rows, run by the
// epilogue warps of the CTA that finished the last head (serve_one's first
// hit, serving.cpp:112-121): warp ballot + prefix over the 8 warps.
// (Visibility of every head's hit/label/prob: the acq_rel arrival that made
// this CTA the last one, then the epilogue barrier.)
__device__ __noinline__ void gap_exit(const TcGapHead& h, int n, int etid, int lane, int* sint) {
  const int warp = etid >> 5;
  int* warp_tot = sint;  // [kEpiWarps]
  int base = 0;
  const unsigned long long now = globaltimer_ns();
  for (int c0 = 0; c0 < n; c0 += kEpiThreads) {
    const int r = c0 + etid;
    const bool valid = r < n;
    const bool hit = valid && __ldcg(h.hit + r) != 0;
    const int id = valid ? h.ids_in[r] : -1;
    if (valid) {
      const int lab = __ldcg(h.label + r);
      if (h.probs_out) h.probs_out[id] = __ldcg(h.prob + r);
      if (h.labels_out) h.labels_out[id] = lab;
      if (hit && h.exit_layer[id] == 0) {
        h.exit_layer[id] = h.layer;
        h.served[id] = lab;
        h.exit_ns[id] = now;
      }
    }
    const bool keep = valid && (h.shadow || !hit);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_tot[warp] = __popc(mask);
    epi_bar();
    int before = 0, total = 0;
    for (int w = 0; w < kEpiWarps; ++w) {
      const int t = warp_tot[w];
      before += w < warp ? t : 0;
      total += t;
    }
    if (keep) {
      const int pos = base + before + __popc(mask & ((1u << lane) - 1u));
      h.ids_out[pos] = id;
      if (h.src_rows_out) h.src_rows_out[pos] = r;
    }
    base += total;
    epi_bar();  // warp_tot reused by the next chunk
  }
  if (etid == 0) {
    *h.count_out = base;
    *h.heads_done = 0;
  }
}

// The GAP features of survivor row r (every tile of the row is complete and
// its partials visible), then the row's cache head when classes > 0.
// fs: >= Cout + 64 floats of shared scratch; sint: >= 64 ints.
__device__ __noinline__ void gap_row_head(const TcConvParams& p, int n, int r, int etid, int lane, float* fs,
                                          int* sint) {
  const TcGapHead& h = p.gh;
  const int img = p.surv ? p.surv[r] : r;
  const float* src = p.gap_out + static_cast<size_t>(img) * p.gap_segs * p.Cout;
  for (int c = etid; c < p.Cout; c += kEpiThreads) {
    float a = 0.0f;
    for (int sg = 0; sg < p.gap_segs; ++sg) a += __ldcg(src + static_cast<size_t>(sg) * p.Cout + c);
    a *= h.inv;
    fs[c] = a;
    if (h.feat) h.feat[static_cast<size_t>(r) * p.Cout + c] = a;
  }
  if (etid == 0) h.row_tiles[r] = 0;  // ready for the next launch
  if (h.classes == 0) return;
  float* lg = fs + p.Cout;  // [32] logits, then [32] pr
  epi_bar();
  const int warp = etid >> 5;
  for (int k = warp; k < h.classes; k += kEpiWarps) {
    const float* wr = h.W2 + static_cast<size_t>(k) * p.Cout;
    float a0 = 0.0f, a1 = 0.0f;
    int c = lane;
    for (; c + 32 < p.Cout; c += 64) {
      a0 += __ldg(wr + c) * fs[c];
      a1 += __ldg(wr + c + 32) * fs[c + 32];
    }
    if (c < p.Cout) a0 += __ldg(wr + c) * fs[c];
    const float a = wsum(a0 + a1);
    if (lane == 0) lg[k] = a + __ldg(h.b2 + k);
  }
  epi_bar();
  if (warp == 0) {
    const bool in = lane < h.classes;
    const float l = in ? lg[lane] : -FLT_MAX;
    const float m = wmax(l);
    const float e = in ? expf(l - m) : 0.0f;
    const float sum = wsum(e);
    const float q = in ? expf(l - m) / sum : 0.0f;
    // argmax(pr), lowest index on ties (tensor.hpp:57-63)
    float bv = in ? q : -FLT_MAX;
    int bi = in ? lane : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    // selector FC(C,16) + ReLU + FC(16,1)
    float z = h.bs2;
    for (int j = 0; j < 16; ++j) {
      const float a = wsum(in ? __ldg(h.Ws1 + j * h.classes + lane) * q : 0.0f) + __ldg(h.bs1 + j);
      z += __ldg(h.ws2 + j) * (a > 0.0f ? a : 0.0f);
    }
    float pz;
    if (z >= 0.0f) {
      pz = 1.0f / (1.0f + expf(-z));
    } else {
      const float ez = expf(z);
      pz = ez / (1.0f + ez);
    }
    if (lane == 0) {
      h.prob[r] = pz;
      h.hit[r] = static_cast<double>(pz) >= h.delta ? 1 : 0;
      h.label[r] = bi;
      sint[63] = atom_add_acq_rel_gpu(h.heads_done, 1) == n - 1 ? 1 : 0;
    }
  }
  epi_bar();
  if (sint[63]) gap_exit(h, n, etid, lane, sint);
}

// One halving step of a 32-value reduce-scatter over the lanes (lanes with
// bit `o` keep the upper kN/2 values and add the partner's): after the steps
// o = 16, 8, 4, 2, 1, lane l holds the full sum of value l.
template <int kN>
__device__ __forceinline__ void rs_half32(float (&v)[32], int o, int lane) {
  const bool up = (lane & o) != 0;
#pragma unroll
  for (int e = 0; e < kN / 2; ++e) {
    const float send = up ? v[e] : v[e + kN / 2];
    const float keep = up ? v[e + kN / 2] : v[e];
    v[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
  }
}

// Post-phase head of survivor row r by ONE warp (classes <= 32): GAP
// features (fixed segment order) -> logits (lane-strided dots of every class,
// reduce-scattered so lane k holds logit k) -> softmax (losses.cpp:35-46) ->
// argmax(pr), lowest index on ties (tensor.hpp:57-63) -> selector
// FC(C,16)+ReLU+FC(16,1) -> branch-stable sigmoid (losses.cpp:26-33) ->
// inclusive p >= delta (cache.cpp:259-265). fs: Cout floats of warp scratch;
// w2s / ws1s: the head weights staged in shared memory by the CTA.
__device__ __noinline__ void row_head_warp(const TcConvParams& p, int r, int lane, float* fs, const float* w2s,
                                           const float* ws1s) {
  const TcGapHead& h = p.gh;
  const int C = p.Cout, K = h.classes, C4 = C >> 2, S = p.gap_segs;
  const int img = p.surv ? p.surv[r] : r;
  const float4* src = reinterpret_cast<const float4*>(p.gap_out + static_cast<size_t>(img) * S * C);
  // lane -> (float4 column j, segment group q of Q): Q = 32 / C4 groups when
  // C < 128 (lanes would idle), each summing segments q, q + Q, ... with four
  // independent accumulators; groups and accumulators combine in fixed order
  const int Q = C4 < 32 ? 32 / C4 : 1;
  for (int j0 = 0; j0 < C4; j0 += 32 / Q) {
    const int j = j0 + (Q > 1 ? lane % C4 : lane), q = Q > 1 ? lane / C4 : 0;
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < C4) {
      int sg = q;
      for (; sg + 3 * Q < S; sg += 4 * Q) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 t = __ldcg(src + static_cast<size_t>(sg + u * Q) * C4 + j);
          a[u].x += t.x;
          a[u].y += t.y;
          a[u].z += t.z;
          a[u].w += t.w;
        }
      }
      for (; sg < S; sg += Q) {
        const float4 t = __ldcg(src + static_cast<size_t>(sg) * C4 + j);
        a[0].x += t.x;
        a[0].y += t.y;
        a[0].z += t.z;
        a[0].w += t.w;
      }
    }
    float4 t = make_float4((a[0].x + a[1].x) + (a[2].x + a[3].x), (a[0].y + a[1].y) + (a[2].y + a[3].y),
                           (a[0].z + a[1].z) + (a[2].z + a[3].z), (a[0].w + a[1].w) + (a[2].w + a[3].w));
    for (int o = C4; o < 32 && Q > 1; o <<= 1) {  // butterfly over the group bits
      t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
      t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
      t.z += __shfl_xor_sync(0xffffffffu, t.z, o);
      t.w += __shfl_xor_sync(0xffffffffu, t.w, o);
    }
    if (j < C4 && q == 0) {
      t = make_float4(t.x * h.inv, t.y * h.inv, t.z * h.inv, t.w * h.inv);
      reinterpret_cast<float4*>(fs)[j] = t;
      if (h.feat) reinterpret_cast<float4*>(h.feat + static_cast<size_t>(r) * C)[j] = t;
    }
  }
  __syncwarp();
  float v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = 0.0f;
#pragma unroll 2
  for (int c = lane; c < C; c += 32) {
    const float f = fs[c];
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < K) v[k] += w2s[k * C + c] * f;
  }
  rs_half32<32>(v, 16, lane);
  rs_half32<16>(v, 8, lane);
  rs_half32<8>(v, 4, lane);
  rs_half32<4>(v, 2, lane);
  rs_half32<2>(v, 1, lane);
  const bool in = lane < K;
  const float l = in ? v[0] + __ldg(h.b2 + lane) : -FLT_MAX;
  const float m = wmax(l);
  const float e = in ? expf(l - m) : 0.0f;
  const float q = e / wsum(e);
  float bv = in ? q : -FLT_MAX;
  int bi = in ? lane : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  // hidden unit j on lane j < 16: bs1[j] + sum_k Ws1[j][k] pr_k (k ascending)
  float hj = 0.0f;
  for (int k = 0; k < K; ++k) {
    const float qk = __shfl_sync(0xffffffffu, q, k);
    if (lane < 16) hj += ws1s[lane * K + k] * qk;
  }
  const float a = lane < 16 ? hj + __ldg(h.bs1 + lane) : 0.0f;
  const float z = h.bs2 + wsum(lane < 16 ? __ldg(h.ws2 + lane) * (a > 0.0f ? a : 0.0f) : 0.0f);
  float pz;
  if (z >= 0.0f) {
    pz = 1.0f / (1.0f + expf(-z));
  } else {
    const float ez = expf(z);
    pz = ez / (1.0f + ez);
  }
  if (lane == 0) {
    h.prob[r] = pz;
    h.hit[r] = static_cast<double>(pz) >= h.delta ? 1 : 0;
    h.label[r] = bi;
  }
}

// Post-phase lookup over the layer's n rows (after the grid barrier): the
// head weights are staged in shared memory, one warp per row across every
// epilogue warp of the grid; each CTA then arrives once and the LAST one runs
// the exit + compaction (gap_exit).
__device__ __noinline__ void post_heads(const TcConvParams& p, int n, int etid, int lane, float* scratch, int* sint) {
  const int ew = etid >> 5;
  const int C = p.Cout, K = p.gh.classes;
  float* w2s = scratch;                                   // [K][C]
  float* ws1s = w2s + K * C;                              // [16][K]
  float* fs = ws1s + 16 * 32 + static_cast<size_t>(ew) * C;  // [kEpiWarps][C]
  const bool any = static_cast<int>(blockIdx.x) < n;  // rows r with r % grid == this CTA
  if (any) {
    for (int i = etid; i < K * C / 4; i += kEpiThreads)
      reinterpret_cast<float4*>(w2s)[i] = __ldg(reinterpret_cast<const float4*>(p.gh.W2) + i);
    for (int i = etid; i < 16 * K; i += kEpiThreads) ws1s[i] = __ldg(p.gh.Ws1 + i);
  }
  epi_bar();
  // rows spread over every CTA first (row r on CTA r % grid, warp r / grid)
  for (int r = blockIdx.x + ew * gridDim.x; r < n; r += gridDim.x * kEpiWarps) row_head_warp(p, r, lane, fs, w2s, ws1s);
  epi_bar();  // this CTA's rows (hit/label/prob) before its arrival
  if (etid == 0) sint[63] = atom_add_acq_rel_gpu(p.gh.heads_done, 1) == static_cast<int>(gridDim.x) - 1 ? 1 : 0;
  epi_bar();
  if (sint[63]) gap_exit(p.gh, n, etid, lane, sint);
}

// After a tile's GAP partials are written by every epilogue warp: count the
// tile against each of its survivor rows; rows completed here get their
// features (and head) from this CTA.
__device__ __noinline__ void gap_complete(const TcConvParams& p, const TileGeom& g, const Tile& x, int etid, int lane,
                                          float* fs, int* sint) {
  epi_bar();  // the tile's GAP partials (every epilogue warp) before the arrivals
  const int ipt = p.halo ? 1 : p.ipt;
  const int target = p.tiles_h * g.tiles_w * g.tiles_n;
  if (etid < ipt) {
    const int idx = x.grp * ipt + etid;
    int r = -1;
    if (idx < g.count && atom_add_acq_rel_gpu(p.gh.row_tiles + idx, 1) == target - 1) r = idx;
    sint[etid] = r;
  }
  epi_bar();
  for (int j = 0; j < ipt; ++j) {
    const int r = sint[j];
    if (r >= 0) gap_row_head(p, g.count, r, etid, lane, fs, sint + 16);
    epi_bar();
  }
}

// Split-K: publish this CTA's partial tile, wait for the other ks-1 CTAs of
// the tile (all resident: one unit per CTA, single round), then reduce 1/ks of
// the tile (warp units of 16 columns x 32 rows, fixed k order) and run the
// epilogue on it. Kept out of line: it is the rare path.
// scratch: >= 8 warps x 2 KB of shared memory (the epilogue staging area).
__device__ __noinline__ bool split_reduce(const TcConvParams& p, const TileGeom& g, const Tile& x, int BN, int etid,
                                          int lane, int unit, uint8_t* scratch, int* last_flag) {
  int* arr = p.ws_counters + 2 * x.tile_mn;
  int* dep = arr + 1;
  const int nu = (BN / 16) * (kBM / 32);
  const int u0 = static_cast<int>((static_cast<long long>(nu) * x.ks) / g.ks);
  const int u1 = static_cast<int>((static_cast<long long>(nu) * (x.ks + 1)) / g.ks);
  const float* tile_ws = p.ws + static_cast<size_t>(x.tile_mn) * g.ks * kBM * BN;
  // wpu warps share a unit (32 rows x 16 columns): warp `sub` sums the
  // partials k in [sub*ks/wpu, (sub+1)*ks/wpu) (all its loads in flight at
  // once), parks the sum in shared memory, and the unit's first warp adds the
  // wpu sums in ascending sub order (fixed association: deterministic).
  const int warp = etid >> 5;
  const int nunits = u1 - u0;
  int wpu = 1;
  while (nunits > 0 && wpu * 2 * nunits <= kEpiWarps) wpu *= 2;  // (a CTA may own no unit: nu < ks)
  const int per_round = kEpiWarps / wpu;
  float4* park = reinterpret_cast<float4*>(scratch);  // [warp][4][32] float4
  // Row geometry (survivor-list load) and BN shift of a round's unit: they do
  // not depend on the partials, so the first round's are fetched between this
  // CTA's arrival and its wait for the others (traced ~3k cycles after the wait otherwise)
  struct RowUnit {
    size_t ob;
    int img;
    bool img_ok, rvalid;
    float4 sh[4];
  };
  auto row_unit = [&](int base, RowUnit& ru) {
    const int uu = base + warp / wpu, sub = warp % wpu;
    const int r = (uu % (kBM / 32)) * 32 + lane;
    const int co = x.tn * BN + (uu / (kBM / 32)) * 16;
    ru.ob = 0;
    ru.img = 0;
    ru.img_ok = false;
    ru.rvalid = false;
    if (uu < u1) {
      ru.rvalid = out_row(p, g, x, r, row_geom(p, r), ru.ob, ru.img, ru.img_ok);
      if (sub == 0 && p.shift) {
#pragma unroll
        for (int q = 0; q < 4; ++q) ru.sh[q] = __ldg(reinterpret_cast<const float4*>(p.shift + co) + q);
      }
    }
  };
  epi_bar();  // this CTA's partial tile stores before the arrival (acq_rel, cumulative)
  if (etid == 0) {
    trace_put(p, unit, 6);
    atom_add_acq_rel_gpu(arr, 1);
  }
  RowUnit ru;
  row_unit(u0, ru);  // while the tile's other CTAs arrive
  if (etid == 0) {
    while (ld_acquire_gpu(arr) < g.ks) __nanosleep(64);
    trace_put(p, unit, 7);
  }
  epi_bar();
  if (etid == 0) trace_put(p, unit, 8);
  for (int base = u0; base < u1; base += per_round) {
    const int uu = base + warp / wpu, sub = warp % wpu;
    const int c16 = uu / (kBM / 32), r = (uu % (kBM / 32)) * 32 + lane;
    const int co = x.tn * BN + c16 * 16;
    if (base != u0) row_unit(base, ru);
    const size_t ob = ru.ob;
    const int img = ru.img;
    const bool img_ok = ru.img_ok, rvalid = ru.rvalid;
    const float4* sh = ru.sh;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.0f;
    if (rvalid) {
      const int k0 = (g.ks * sub) / wpu, k1 = (g.ks * (sub + 1)) / wpu;
#pragma unroll 6  // the partial loads of 6 k's go out together; the adds keep ascending k order
      for (int k = k0; k < k1; ++k) {
        // layout [k][c16][q][row] float4: a warp's load of one q is 512 contiguous bytes
        const float4* src = reinterpret_cast<const float4*>(tile_ws + static_cast<size_t>(k) * kBM * BN) +
                            static_cast<size_t>(c16) * 4 * kBM + r;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 f = __ldcg(src + u * kBM);
          v[4 * u] += f.x;
          v[4 * u + 1] += f.y;
          v[4 * u + 2] += f.z;
          v[4 * u + 3] += f.w;
        }
      }
    }
    TC_TRACE(if (warp == 0 && lane == 0 && base == u0) trace_val(p, unit, 15, clk());)
    if (wpu > 1) {
      if (uu < u1) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          park[(warp * 4 + u) * 32 + lane] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
      }
      epi_bar();
    }
    if (uu < u1 && sub == 0) {
      if (rvalid) {
        for (int w = 1; w < wpu; ++w) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 f = park[((warp + w) * 4 + u) * 32 + lane];
            v[4 * u] += f.x;
            v[4 * u + 1] += f.y;
            v[4 * u + 2] += f.z;
            v[4 * u + 3] += f.w;
          }
        }
        uint4 rh[2], rl[2];
        if (p.res_hi) {
          rh[0] = reinterpret_cast<const uint4*>(p.res_hi + ob + co)[0];
          rh[1] = reinterpret_cast<const uint4*>(p.res_hi + ob + co)[1];
          if (p.res_lo) {
            rl[0] = reinterpret_cast<const uint4*>(p.res_lo + ob + co)[0];
            rl[1] = reinterpret_cast<const uint4*>(p.res_lo + ob + co)[1];
          }
        }
        epilogue_math(p, v, co, p.shift ? reinterpret_cast<const float*>(sh) : nullptr, p.res_hi ? rh : nullptr,
                      p.res_lo ? rl : nullptr);
        uint4 hi[2], lo[2];
        split16(v, hi, lo);
        uint4* oh = reinterpret_cast<uint4*>(p.out_hi + ob + co);
        oh[0] = hi[0];
        oh[1] = hi[1];
        if (p.out_lo) {
          uint4* ol = reinterpret_cast<uint4*>(p.out_lo + ob + co);
          ol[0] = lo[0];
          ol[1] = lo[1];
        }
        TC_TRACE(if (warp == 0 && lane == 0 && base == u0) trace_val(p, unit, 12, clk());)
      }
      if (p.gap_out) gap_segment(p, x, r, lane, v, co, img, img_ok);  // v = 0 on rows outside the output
      if (lane == 0) trace_put(p, unit, 9 + (warp < 2 ? warp : 1));
    }
    if (wpu > 1) epi_bar();  // park slots reused by the next round
  }
  if (etid == 0) trace_put(p, unit, 11);
  // the next split-K launch zeroes this counter set (post-phase lookups need no per-tile completion)
  if (p.ctr_zero && (!p.gh.row_tiles || p.gh.post)) return false;
  epi_bar();  // this CTA's GAP partials visible before its arrival
  if (etid == 0) {
    const bool last = atom_add_acq_rel_gpu(dep, 1) == g.ks - 1;
    if (last) {
      *arr = 0;
      *dep = 0;
    }
    *last_flag = last ? 1 : 0;
  }
  epi_bar();
  return *last_flag != 0;
}

template <int BN, bool X3>
__global__ void __launch_bounds__(kThreads, 1) tc_conv_kernel(const __grid_constant__ TcConvParams p) {
  using Cfg = TcCfg<BN, X3>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base for the swizzled operands, derived by offsetting
  // the __shared__ array itself so the compiler keeps the shared address space
  // (plain C++ accesses, e.g. the epilogue's shift values, become LDS rather
  // than generic loads through the global path)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // stage s: [A_hi][A_lo?][B_hi][B_lo?]
  // barriers: [0,8) full (stages / halo B ring), [8,16) empty, [16,18) tfull,
  // [18,20) tempty, [20,22) halo A-slab full, [22,24) halo A-slab empty
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes + Cfg::kEpiStage);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 32);
  float* shift_s = reinterpret_cast<float*>(smem + S * Cfg::kStageBytes + Cfg::kEpiStage + 1024);  // [2][BN]
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = smem_u32(bars + 8);
  const uint32_t tfull0 = smem_u32(bars + 16);
  const uint32_t tempty0 = smem_u32(bars + 18);
  const uint32_t afull0 = smem_u32(bars + 20);
  const uint32_t aempty0 = smem_u32(bars + 22);
  // per epilogue warp TMA-store staging (after the pipeline stages; bars follow)
  uint8_t* epi_stage = smem + S * Cfg::kStageBytes;
  auto stage_a = [&](int s, int plane) { return smem + s * Cfg::kStageBytes + plane * kABytes; };
  auto stage_b = [&](int s, int plane) {
    return smem + s * Cfg::kStageBytes + Cfg::kPlanes * kABytes + plane * Cfg::kBBytes;
  };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace_put(p, 0, 26);  // CTA entry
  // debug bits (measurement only): 1 = no TMA loads, 2 = no MMAs, 4 = no epilogue stores
  const bool dbg_noload = (p.dbg & 1) != 0, dbg_nomma = (p.dbg & 2) != 0, dbg_nostore = (p.dbg & 4) != 0;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 8; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(afull0 + 8 * i, 1);
      mbar_init(aempty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull0 + 8 * i, 1);
      mbar_init(tempty0 + 8 * i, kEpiWarps);
    }
    fence_mbar_init();
    tma_prefetch_desc(&p.tmA[0]);
    tma_prefetch_desc(&p.tmB[0]);
    if (X3) {
      tma_prefetch_desc(&p.tmA[1]);
      tma_prefetch_desc(&p.tmB[1]);
    }
    if (p.nres) {
      tma_prefetch_desc(&p.tmR[0]);
      if (X3) tma_prefetch_desc(&p.tmR[1]);
      if (p.res_proj) {
        tma_prefetch_desc(&p.tmP[0]);
        if (X3) tma_prefetch_desc(&p.tmP[1]);
      } else {
        tma_prefetch_desc(&p.tmE);
      }
    }
  }
  if (warp == 0) tmem_alloc(smem_u32(tmem_holder), Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) trace_put(p, 0, 27);  // barriers + TMEM ready
  // weights do not depend on upstream kernels: warm L2 with this CTA's share
  // while the previous kernel drains (short split-K units otherwise wait on
  // first-touch HBM latency for every B box)
  if (warp == 0 && p.wpre_bytes > 0) {
    // (32-bit division: weight planes are < 2^31 bytes)
    const long long chunk =
        ((static_cast<unsigned>(p.wpre_bytes) + gridDim.x - 1) / gridDim.x + 15) & ~15LL;
    const long long off = static_cast<long long>(blockIdx.x) * chunk;
    if (off < p.wpre_bytes) {
      const long long len = p.wpre_bytes - off < chunk ? p.wpre_bytes - off : chunk;
      if (lane < (X3 ? 2 : 1) && p.wpre[lane]) {
        const char* base = static_cast<const char*>(p.wpre[lane]) + off;
        for (long long o = 0; o < len; o += 65536) {
          const unsigned n = static_cast<unsigned>(len - o < 65536 ? len - o : 65536);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(n) : "memory");
        }
      }
    }
  }
  // everything above is independent of upstream kernels (programmatic launch)
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) trace_put(p, 0, 28);  // upstream complete
  if (p.ctr_zero && threadIdx.x == 0)
    for (int i = blockIdx.x; i < p.ctr_len; i += gridDim.x) p.ctr_zero[i] = 0;

  const TileGeom g = tile_geom(p, BN);
  const int cchunks = p.C / 64;
  // fused lookup with no rows: nobody finishes a head, so the compaction count is written here
  if (p.gh.row_tiles && p.gh.classes && g.count == 0 && blockIdx.x == 0 && threadIdx.x == 0) *p.gh.count_out = 0;
  int* const sint = reinterpret_cast<int*>(bars + 64);  // 64 ints of epilogue flags (in the barrier block)
  const int cs = p.conv_stride > 0 ? p.conv_stride : 1;

  // halo mode ring carving (runtime): A-slab slots then B slots inside the stage region
  const uint32_t ring0 = smem_u32(smem);
  const uint32_t h_aslot = static_cast<uint32_t>(Cfg::kPlanes) * p.halo_aplane;
  const uint32_t h_bslot = static_cast<uint32_t>(Cfg::kPlanes) * Cfg::kBBytes;
  const uint32_t h_b0 = ring0 + 2u * h_aslot;
  const int h_sb = p.halo_sb;

  if (warp == 0 && p.halo) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (halo)
      // Per 64-channel chunk one slab of padded rows (box {64, Pw, rows}) feeds
      // all k*k taps; per (chunk, tap) one weight tile into the B ring.
      int aslot = 0, bslot = 0;
      uint32_t aphase = 0, bphase = 0;
      const int nk_conv = p.ntaps * cchunks;
      const int pad = -p.tap_dw[0];
      const uint32_t a_bytes = static_cast<uint32_t>(Cfg::kPlanes * p.halo_pw * p.halo_rows * 128);
      const uint32_t r_bytes = static_cast<uint32_t>(Cfg::kPlanes * p.halo_pw * p.halo_res_rows * 128);
      int unit = 0;
      for (int t = blockIdx.x; t < g.total; t += gridDim.x, ++unit) {
        const Tile x = decode_tile(t, p, g);
        trace_put(p, unit, 0);
        const int img = image_of(p, x.grp < g.count ? x.grp : g.count - 1);
        const int m0 = x.h0 * kBM;
        const int R0 = m0 / p.halo_pw;
        for (int s = x.s_begin; s < x.s_end; ++s) {
          const bool res = s >= nk_conv;
          const int cc = res ? 0 : s / p.ntaps, tap = res ? 0 : s % p.ntaps;
          if (res || tap == 0 || s == x.s_begin) {
            mbar_wait(aempty0 + 8 * aslot, aphase ^ 1);
            const uint32_t fb = afull0 + 8 * aslot;
            mbar_expect_tx(fb, dbg_noload ? 0u : (res ? r_bytes : a_bytes));
            if (!dbg_noload)
            for (int pl = 0; pl < Cfg::kPlanes; ++pl) {
              const uint32_t dst = ring0 + aslot * h_aslot + pl * p.halo_aplane;
              if (res)
                tma_load_5d(dst, &p.tmR[pl], fb, x.tn * BN + (s - nk_conv) * 64, 0, R0, img, 0);
              else
                tma_load_5d(dst, &p.tmA[pl], fb, cc * 64, -pad, R0 - pad, img, 0);
            }
            if (res || tap == p.ntaps - 1 || s == x.s_end - 1) {
              if (++aslot == 2) {
                aslot = 0;
                aphase ^= 1;
              }
            }
          } else if (tap == p.ntaps - 1 || s == x.s_end - 1) {
            if (++aslot == 2) {
              aslot = 0;
              aphase ^= 1;
            }
          }
          mbar_wait(empty0 + 8 * bslot, bphase ^ 1);
          const uint32_t fb = full0 + 8 * bslot;
          mbar_expect_tx(fb, dbg_noload ? 0u : static_cast<uint32_t>(Cfg::kPlanes * Cfg::kBBytes));
          for (int pl = 0; pl < (dbg_noload ? 0 : Cfg::kPlanes); ++pl) {
            const uint32_t dst = h_b0 + bslot * h_bslot + pl * Cfg::kBBytes;
            if (res)
              tma_load_2d(dst, &p.tmE, fb, (s - nk_conv) * 64, 0);
            else
              tma_load_2d(dst, &p.tmB[pl], fb, tap * p.C + cc * 64, x.tn * BN);
          }
          if (++bslot == h_sb) {
            bslot = 0;
            bphase ^= 1;
          }
        }
        trace_put(p, unit, 1);
      }
    }
  } else if (warp == 1 && p.halo) {
    {  // whole warp: uniform operands, elect.sync issues
      // ------------------------------------------------ MMA issuer (halo)
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
      constexpr uint32_t idesc2 = umma_idesc_bf16(kBM, X3 ? 2 * BN : BN);  // stacked [B_hi; B_lo]
      const bool stacked = X3 && p.stacked != 0;
      int aslot = 0, bslot = 0;
      uint32_t aphase = 0, bphase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const int nk_conv = p.ntaps * cchunks;
      const int kk = p.tap_dw[p.ntaps - 1] - p.tap_dw[0] + 1;  // filter width
      int unit = 0;
      for (int t = blockIdx.x; t < g.total; t += gridDim.x, ++unit) {
        const Tile x = decode_tile(t, p, g);
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0) trace_put(p, unit, 2);
        const uint32_t d_tmem = tmem_base + acc * Cfg::kAccCols;
        const int m0 = x.h0 * kBM;
        const int base_row = m0 - (m0 / p.halo_pw) * p.halo_pw;  // anchor m0 inside the slab
        for (int s = x.s_begin; s < x.s_end; ++s) {
          const bool res = s >= nk_conv;
          const int tap = res ? 0 : s % p.ntaps;
          const bool new_a = res || tap == 0 || s == x.s_begin;
          const bool last_a = res || tap == p.ntaps - 1 || s == x.s_end - 1;
          if (new_a) mbar_wait(afull0 + 8 * aslot, aphase);
          mbar_wait(full0 + 8 * bslot, bphase);
          tc_fence_after();
          int row_off = res ? base_row : base_row + (tap / kk) * p.halo_pw + (tap % kk);
          if (p.dbg & 8) row_off &= ~7;  // measurement only: 8-row-aligned operand starts (wrong values)
          const uint32_t ah = ring0 + aslot * h_aslot + static_cast<uint32_t>(row_off) * 128;
          const uint32_t al = ah + p.halo_aplane;
          const uint32_t bh = h_b0 + bslot * h_bslot, bl = bh + Cfg::kBBytes;
// (a runtime trip count here miscompiles the MMA sequence: keep it constant)
          // K-advance of 16 bf16 = 32 bytes = +2 in the descriptor's address field
          const uint64_t dah = umma_desc_sw128(ah), dal = umma_desc_sw128(al);
          const uint64_t dbh = umma_desc_sw128(bh), dbl = umma_desc_sw128(bl);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (dbg_nomma) break;
            const uint32_t first = (s > x.s_begin || k > 0) ? 1u : 0u;
            if (stacked && !res) {  // [hi*hi | hi*lo] in one MMA, then lo*hi into the low half
              umma_bf16_warp(d_tmem, dah + 2 * k, dbh + 2 * k, idesc2, first);
              umma_bf16_warp(d_tmem, dal + 2 * k, dbh + 2 * k, idesc, 1u);
            } else {
              umma_bf16_warp(d_tmem, dah + 2 * k, dbh + 2 * k, idesc, first);
              if (X3) {
                if (!res) umma_bf16_warp(d_tmem, dah + 2 * k, dbl + 2 * k, idesc, 1u);
                umma_bf16_warp(d_tmem, dal + 2 * k, dbh + 2 * k, idesc, 1u);
              }
            }
          }
          umma_commit_warp(empty0 + 8 * bslot);
          if (++bslot == h_sb) {
            bslot = 0;
            bphase ^= 1;
          }
          if (last_a) {
            umma_commit_warp(aempty0 + 8 * aslot);
            if (++aslot == 2) {
              aslot = 0;
              aphase ^= 1;
            }
          }
        }
        umma_commit_warp(tfull0 + 8 * acc);
        if (lane == 0) trace_put(p, unit, 3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp == 0) {
    {
      // ------------------------------------------------ TMA producer (whole warp)
      // A stage's TMA boxes (per plane: nbox activation boxes + one weight
      // box) are spread over the lanes and issued by one warp instruction: a
      // single thread issuing them back to back is latency-bound (~2x slower
      // on the 5-D activation boxes, tests/cuda/tma_lat.cu).
      int stage = 0;
      uint32_t phase = 0;
      const int box_bytes = p.hb * p.wb * 128;
      int unit = 0;
      for (int t = blockIdx.x; t < g.total; t += gridDim.x, ++unit) {
        const Tile x = decode_tile(t, p, g);
        if (lane == 0) trace_put(p, unit, 0);
        const int ipt = p.plain ? 1 : p.ipt;
        // lane j < ipt: image of the tile's j-th slot (rows of missing slots are discarded by the epilogue)
        int my_img = 0;
        if (!p.plain && lane < ipt) {
          int idx = x.grp * ipt + lane;
          if (idx >= g.count) idx = g.count - 1;
          my_img = image_of(p, idx);
        }
        const int img0 = __shfl_sync(0xffffffffu, my_img, 0);
        // one box for all ipt images when their ids are consecutive
        const bool consec = p.multi_img != 0 && ipt > 1 && x.grp * ipt + ipt <= g.count &&
                            __all_sync(0xffffffffu, lane >= ipt || my_img == img0 + lane);
        const CUtensorMap* mapA = consec ? p.tmAm : p.tmA;
        const CUtensorMap* mapR = consec ? p.tmRm : p.tmR;
        const int nbox = consec ? 1 : ipt;
        // this lane's task in every stage: plane pl, box j (j == nbox: the B box)
        // (tiles of tiny images, up to 16 per tile with scattered ids, have up to
        // 34 tasks: lanes take tasks lane and lane + 32)
        const int ntask = Cfg::kPlanes * (nbox + 1);
        const int pl = lane / (nbox + 1), jb = lane % (nbox + 1);
        const int img_j = __shfl_sync(0xffffffffu, my_img, jb < nbox ? jb : 0);
        const int pl2 = (lane + 32) / (nbox + 1), jb2 = (lane + 32) % (nbox + 1);
        const int img_j2 = __shfl_sync(0xffffffffu, my_img, jb2 < nbox && jb2 < 32 ? jb2 : 0);
        const int nk_conv = p.ntaps * cchunks;
        // residual K-step j: A box coordinates (channel, w, h) and B box (k, n)
        const int rs = p.res_stride > 0 ? p.res_stride : 1;
        const int rc0 = p.res_proj ? 0 : x.tn * BN, rw = x.w0 * rs, rh = x.h0 * rs;
        const CUtensorMap* mapE = p.res_proj ? p.tmP : &p.tmE;  // plane q: mapE[res_proj ? q : 0]
        const int en = p.res_proj ? x.tn * BN : 0;
        int cc = x.s_begin % cchunks, tap = x.s_begin / cchunks;
        TC_TRACE(unsigned long long pw = 0;)  // cycles spent waiting for free stages
        for (int s = x.s_begin; s < x.s_end; ++s) {
          TC_TRACE(const unsigned long long c0 = p.trace ? clk() : 0;)
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          TC_TRACE(if (p.trace) pw += clk() - c0;)
          const uint32_t fb = full0 + 8 * stage;
          if (lane == 0) mbar_expect_tx(fb, dbg_noload ? 0u : static_cast<uint32_t>(Cfg::kStageBytes));
          __syncwarp();
          if (!dbg_noload && ntask <= 32 && lane < ntask) {
            const uint32_t a_dst = smem_u32(stage_a(stage, pl)) + jb * box_bytes;
            if (s >= nk_conv) {
              // residual K-step: A = residual channels [tn*BN + j*64, +64) at the
              // output pixels, B = identity slice (the residual add on the tensor
              // core); fused projection: A = block-input channels [j*64, +64) at
              // stride res_stride, B = projection weights [tn*BN, +BN) x [j*64, +64)
              const int j = s - nk_conv;
              if (jb < nbox)
                tma_load_5d(a_dst, &mapR[pl], fb, rc0 + j * 64, rw, rh, img_j, 0);
              else
                tma_load_2d(smem_u32(stage_b(stage, pl)), &mapE[p.res_proj ? pl : 0], fb, j * 64, en);
            } else {
              if (jb < nbox) {
                const int wc = x.w0 * cs + p.tap_dw[tap], hc = x.h0 * cs + p.tap_dh[tap], ph = p.tap_phase[tap];
                tma_load_5d(a_dst, &mapA[pl], fb, cc * 64, wc, hc, img_j, ph);
              } else {
                tma_load_2d(smem_u32(stage_b(stage, pl)), &p.tmB[pl], fb, tap * p.C + cc * 64, x.tn * BN);
              }
            }
          } else if (!dbg_noload && ntask > 32) {
            // tiny images (> 15 per tile) with scattered ids: tasks lane and lane + 32
            for (int tk = lane; tk < ntask; tk += 32) {
              const int plx = tk < 32 ? pl : pl2, jbx = tk < 32 ? jb : jb2, imgx = tk < 32 ? img_j : img_j2;
              const uint32_t a_dst = smem_u32(stage_a(stage, plx)) + jbx * box_bytes;
              if (s >= nk_conv) {
                const int j = s - nk_conv;
                if (jbx < nbox)
                  tma_load_5d(a_dst, &mapR[plx], fb, rc0 + j * 64, rw, rh, imgx, 0);
                else
                  tma_load_2d(smem_u32(stage_b(stage, plx)), &mapE[p.res_proj ? plx : 0], fb, j * 64, en);
              } else if (jbx < nbox) {
                tma_load_5d(a_dst, &mapA[plx], fb, cc * 64, x.w0 * cs + p.tap_dw[tap], x.h0 * cs + p.tap_dh[tap], imgx,
                            p.tap_phase[tap]);
              } else {
                tma_load_2d(smem_u32(stage_b(stage, plx)), &p.tmB[plx], fb, tap * p.C + cc * 64, x.tn * BN);
              }
            }
          }
          if (++cc == cchunks) {
            cc = 0;
            ++tap;
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) trace_put(p, unit, 1);
        TC_TRACE(if (lane == 0) trace_val(p, unit, 14, pw);)
      }
    }
  } else if (warp == 1) {
    {  // whole warp: uniform operands, elect.sync issues
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
      constexpr uint32_t idesc2 = umma_idesc_bf16(kBM, X3 ? 2 * BN : BN);  // stacked [B_hi; B_lo]
      const bool stacked = X3 && p.stacked != 0;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int unit = 0;
      const uint64_t dah0 = umma_desc_sw128(smem_u32(stage_a(0, 0))), dbh0 = umma_desc_sw128(smem_u32(stage_b(0, 0)));
      const uint64_t dal0 = umma_desc_sw128(smem_u32(stage_a(0, X3 ? 1 : 0)));
      const uint64_t dbl0 = umma_desc_sw128(smem_u32(stage_b(0, X3 ? 1 : 0)));
      for (int t = blockIdx.x; t < g.total; t += gridDim.x, ++unit) {
        const Tile x = decode_tile(t, p, g);
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0) trace_put(p, unit, 2);
        const uint32_t d_tmem = tmem_base + acc * Cfg::kAccCols;
        const int nk_conv = p.ntaps * (p.C / 64);
        TC_TRACE(unsigned long long mw = 0, mi = 0;)  // cycles waiting for data / issuing + committing
        for (int s = x.s_begin; s < x.s_end; ++s) {
          TC_TRACE(const unsigned long long c0 = p.trace ? clk() : 0;)
          mbar_wait(full0 + 8 * stage, phase);
          tc_fence_after();
          TC_TRACE(const unsigned long long c1 = p.trace ? clk() : 0;)
          // identity K-step (residual add); a fused projection's K-steps are
          // ordinary bf16x3 K-steps (three products, low accumulator half)
          const bool res_step = s >= nk_conv && !p.res_proj;
          const bool proj_step = s >= nk_conv && p.res_proj;
          // K-advance of 16 bf16 = 32 bytes = +2 in the descriptor's address
          // field; stage k's operands sit k * kStageBytes further (< 256 KB,
          // so the 14-bit address field never carries)
          const uint64_t so = static_cast<uint64_t>(stage) * (Cfg::kStageBytes >> 4);
          const uint64_t dah = dah0 + so, dbh = dbh0 + so, dal = dal0 + so, dbl = dbl0 + so;
          // whole K-steps under one elect.sync (the MMA warp is issue-bound);
          // LCB_DBG bit 16 keeps the per-MMA path for A/B measurements
          const bool fused_issue = !dbg_nomma && !(p.dbg & 16);
          const uint32_t eb = empty0 + 8 * stage;
          if (fused_issue && stacked && !res_step && !proj_step) {
            umma_kstep_x3_stacked(d_tmem, dah, dal, dbh, idesc2, idesc, s > x.s_begin ? 1u : 0u, eb);
          } else if (fused_issue && X3 && !res_step) {
            umma_kstep_x3_plain(d_tmem, dah, dal, dbh, dbl, idesc, s > x.s_begin ? 1u : 0u, eb);
          } else if (fused_issue && X3 && res_step) {
            umma_kstep_x3_res(d_tmem, dah, dal, dbh, idesc, s > x.s_begin ? 1u : 0u, eb);
          } else if (fused_issue && !X3) {
            umma_kstep_bf16(d_tmem, dah, dbh, idesc, s > x.s_begin ? 1u : 0u, eb);
          } else {
// (a runtime trip count here miscompiles the MMA sequence: keep it constant)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (dbg_nomma) break;
            const uint32_t first = (s > x.s_begin || k > 0) ? 1u : 0u;
            if (stacked && !res_step && !proj_step) {  // [hi*hi | hi*lo] in one MMA, then lo*hi into the low half
              umma_bf16_warp(d_tmem, dah + 2 * k, dbh + 2 * k, idesc2, first);
              umma_bf16_warp(d_tmem, dal + 2 * k, dbh + 2 * k, idesc, 1u);
            } else {
              umma_bf16_warp(d_tmem, dah + 2 * k, dbh + 2 * k, idesc, first);
              if (X3) {
                if (!res_step)  // identity has no lo plane
                  umma_bf16_warp(d_tmem, dah + 2 * k, dbl + 2 * k, idesc, 1u);
                umma_bf16_warp(d_tmem, dal + 2 * k, dbh + 2 * k, idesc, 1u);
              }
            }
          }
          umma_commit_warp(eb);
          }
          TC_TRACE(if (p.trace) {
            mw += c1 - c0;
            mi += clk() - c1;
          })
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_warp(tfull0 + 8 * acc);
        if (lane == 0) trace_put(p, unit, 3);
        TC_TRACE(if (lane == 0) {
          trace_val(p, unit, 12, mw);
          trace_val(p, unit, 13, mi);
        })
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------ epilogue
    // warp w: TMEM lane quadrant w % 4 (tile rows), column half (w - 2) / 4;
    // 32 columns per step: TMEM -> registers -> shift / residual / ReLU ->
    // hi/lo -> shared staging (64-byte swizzle) -> 8 rows x 64 contiguous
    // bytes per store instruction. Rolled loops keep the code small (the MMA
    // and TMA warps share the instruction cache with this code).
    constexpr int kCols = BN / 2;  // columns per epilogue warp
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const int etid = threadIdx.x - 64;  // 0..255
    const int col0 = half * kCols;
    const uint32_t wstage = smem_u32(epi_stage + (warp - 2) * Cfg::kEpiWarpBytes);
    int acc = 0;
    uint32_t acc_phase = 0;
    int unit = 0;
    // the output row of the NEXT tile is resolved one tile ahead (its
    // survivor-id load then overlaps this tile's epilogue)
    size_t obase_n = 0;
    bool valid_n = false, img_ok_n = false;
    int img_n = 0;
    const RowGeom rg = row_geom(p, row);
    // per-tile shift values live in shared memory, double-buffered with the
    // accumulators; the NEXT tile's values are loaded into registers while
    // this tile is processed (their L2 latency was a serial gap per tile)
    // (reading them from global memory without the per-tile barrier measured slower)
    const bool use_shs = p.shift && p.mode == 0;
    static_assert(BN <= kEpiThreads, "one shift value per epilogue thread");
    if (static_cast<int>(blockIdx.x) < g.total) {
      const Tile x0 = decode_tile(blockIdx.x, p, g);
      valid_n = out_row(p, g, x0, row, rg, obase_n, img_n, img_ok_n);
      if (use_shs && etid < BN) shift_s[etid] = __ldg(p.shift + x0.tn * BN + etid);
    }
    for (int t = blockIdx.x; t < g.total; t += gridDim.x, ++unit) {
      const Tile x = decode_tile(t, p, g);
      const size_t obase = obase_n;
      const bool valid = valid_n, img_ok = img_ok_n;
      const int img = img_n;
      const bool has_next = t + static_cast<int>(gridDim.x) < g.total;
      float nsh = 0.0f;
      if (has_next) {
        const Tile xn = decode_tile(t + gridDim.x, p, g);
        valid_n = out_row(p, g, xn, row, rg, obase_n, img_n, img_ok_n);
        if (use_shs && etid < BN) nsh = __ldg(p.shift + xn.tn * BN + etid);
      }
      const bool split = p.mode == 0 && g.ks > 1;
      // this tile's shift values (written at the end of the previous tile, or
      // before the loop); the barrier also retires every warp's reads of the
      // other buffer (tile t-1), which the end of this tile overwrites
      float* shs = shift_s + acc * BN;
      if (use_shs) epi_bar();
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      if (etid == 0) trace_put(p, unit, 4);
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * Cfg::kAccCols + col0;
      const bool empty_k = x.s_end <= x.s_begin;  // no MMA wrote this accumulator
      // stacked: the hi*lo half holds data only if a conv K-step initialised it
      const bool upper = X3 && p.stacked != 0 && x.s_begin < p.ntaps * (p.C / 64);
      // rows this lane stores in the coalesced phase (lane/4 + 8i of the warp's 32)
      size_t st_ob[4];
      bool st_ok[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = (lane >> 2) + 8 * i;
        st_ob[i] = __shfl_sync(0xffffffffu, static_cast<unsigned long long>(obase), r);
        st_ok[i] = __shfl_sync(0xffffffffu, valid ? 1 : 0, r) != 0;
      }
      // split-K partial tile layout: [tile_mn][ks][BN/16][4 float4 groups][128 rows] (coalesced per warp)
      float* wsp = split ? p.ws + (static_cast<size_t>(x.tile_mn) * g.ks + x.ks) * kBM * BN : nullptr;
#pragma unroll kEpiUnroll
      for (int c32 = 0; c32 < kCols / 32; ++c32) {
        float v[2][16];
        tmem_ld16_nowait(t_row + c32 * 32, v[0]);
        tmem_ld16_nowait(t_row + c32 * 32 + 16, v[1]);
        if (upper) {
          float w[2][16];
          tmem_ld16_nowait(t_row + BN + c32 * 32, w[0]);
          tmem_ld16_nowait(t_row + BN + c32 * 32 + 16, w[1]);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            v[0][i] += w[0][i];
            v[1][i] += w[1][i];
          }
        } else {
          tmem_ld_wait();
        }
        TC_TRACE(if (etid == 0 && c32 < 2) trace_put(p, unit, 16 + 4 * c32);)
        const int cb = x.tn * BN + col0 + c32 * 32;  // first output channel of this step
        if (empty_k) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[0][i] = v[1][i] = 0.0f;
        }
        if (split) {
          if (valid) {  // the reduction reads valid rows only
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int c16 = (col0 >> 4) + c32 * 2 + u;
              float4* dst = reinterpret_cast<float4*>(wsp) + static_cast<size_t>(c16) * 4 * kBM + row;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                __stcg(dst + q * kBM, make_float4(v[u][4 * q], v[u][4 * q + 1], v[u][4 * q + 2], v[u][4 * q + 3]));
            }
          }
          continue;
        }
        if (p.mode == 1 || (p.mix_n1 > 0 && x.tn * BN >= p.mix_n1)) {
          if (valid) {
            const int f32_ld = p.mix_n1 > 0 ? p.mix_ld : p.Cout;
            float* dst = p.out_f32 + (static_cast<size_t>(x.ks) * p.rows_total + x.w0 + row) * f32_ld + (cb - p.mix_n1);
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int q = 0; q < 4; ++q)
                reinterpret_cast<float4*>(dst + u * 16)[q] =
                    make_float4(v[u][4 * q], v[u][4 * q + 1], v[u][4 * q + 2], v[u][4 * q + 3]);
          }
          continue;
        }
        // mode 0: epilogue math, staged coalesced store, fused GAP partials
        __syncwarp();  // previous step's staging read back
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int co = cb + u * 16;
          uint4 rh[2], rl[2];
          const bool r = valid && p.res_hi;  // epilogue residual (LCB_NO_MMA_RESIDUAL); default adds it on the MMA
          if (r) {
            rh[0] = reinterpret_cast<const uint4*>(p.res_hi + obase + co)[0];
            rh[1] = reinterpret_cast<const uint4*>(p.res_hi + obase + co)[1];
            if (X3 && p.res_lo) {
              rl[0] = reinterpret_cast<const uint4*>(p.res_lo + obase + co)[0];
              rl[1] = reinterpret_cast<const uint4*>(p.res_lo + obase + co)[1];
            }
          }
          epilogue_math(p, v[u], co, p.shift ? shs + (co - x.tn * BN) : nullptr, r ? rh : nullptr,
                        (r && X3 && p.res_lo) ? rl : nullptr);
          if (!valid && p.gap_out) {  // (stores skip invalid rows; the GAP partials need zeros there)
#pragma unroll
            for (int i = 0; i < 16; ++i) v[u][i] = 0.0f;
          }
          uint4 hi[2], lo[2];
          split16(v[u], hi, lo);
#pragma unroll
          for (int hq = 0; hq < 2; ++hq) {
            const uint32_t off = static_cast<uint32_t>(lane * 64 + (((u * 2 + hq) ^ ((lane >> 1) & 3)) * 16));
            st_shared_v4(wstage + off, hi[hq]);
            if (X3) st_shared_v4(wstage + 2048 + off, lo[hq]);
          }
        }
        TC_TRACE(if (etid == 0 && c32 < 2) trace_put(p, unit, 17 + 4 * c32);)
        __syncwarp();
        {
          const int ch = lane & 3;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = (lane >> 2) + 8 * i;  // row within the warp
            const uint32_t off = static_cast<uint32_t>(r * 64 + ((ch ^ ((r >> 1) & 3)) * 16));
            if (st_ok[i] && !dbg_nostore) {
              *reinterpret_cast<uint4*>(p.out_hi + st_ob[i] + cb + ch * 8) = ld_shared_v4(wstage + off);
              if (X3 && p.out_lo)
                *reinterpret_cast<uint4*>(p.out_lo + st_ob[i] + cb + ch * 8) = ld_shared_v4(wstage + 2048 + off);
            }
          }
        }
        TC_TRACE(if (etid == 0 && c32 < 2) trace_put(p, unit, 18 + 4 * c32);)
        if (p.gap_out) {
          gap_segment(p, x, row, lane, v[0], cb, img, img_ok);  // destroys v (after staging)
          gap_segment(p, x, row, lane, v[1], cb + 16, img, img_ok);
        }
      }
      if (use_shs && has_next && etid < BN) shift_s[(acc ^ 1) * BN + etid] = nsh;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      const bool per_tile = p.gh.row_tiles && !p.gh.post;
      if (split) {
        if (split_reduce(p, g, x, BN, etid, lane, unit, epi_stage, sint + 127) && per_tile)
          gap_complete(p, g, x, etid, lane, reinterpret_cast<float*>(epi_stage), sint);
      } else if (per_tile) {
        gap_complete(p, g, x, etid, lane, reinterpret_cast<float*>(epi_stage), sint);
      }
      if (etid == 0) trace_put(p, unit, 5);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_put(p, 0, 29);  // all roles done
  if (warp == 0) {
    __syncwarp();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
  if (p.gh.row_tiles && p.gh.post && !(p.dbg & 64)) {  // (dbg 64/32: measurement only, no post-phase / no heads)
    // Lookup post-phase: every CTA's GAP partials are written; one grid
    // barrier, then the survivor rows' features and heads (row-strided over
    // the CTAs, epilogue warps), the last head's CTA runs exit + compaction.
    // Monotonic counter: each launch adds kPostSyncPeriod in total (gridDim.x
    // arrivals, CTA 0 pads), so its base is the counter rounded down.
    constexpr unsigned kPostSyncPeriod = 256;  // >= grid, divides 2^32
    if (threadIdx.x == 0) {
      const unsigned base = ld_acquire_u32(p.gh.gsync) & ~(kPostSyncPeriod - 1u);
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.gh.gsync) : "memory");
      while (ld_acquire_u32(p.gh.gsync) - base < gridDim.x) __nanosleep(32);
      if (blockIdx.x == 0)
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p.gh.gsync), "r"(kPostSyncPeriod - gridDim.x)
                     : "memory");
    }
    __syncthreads();
    if (warp >= 2 && !(p.dbg & 32))  // the (idle) pipeline stages are the warps' feature scratch
      post_heads(p, g.count, threadIdx.x - 64, lane, reinterpret_cast<float*>(smem), sint);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
  }
  return fn;
}

template <int BN, bool X3>
cudaError_t launch_cfg(const TcConvParams& p, int num_sms, cudaStream_t stream) {
  using Cfg = TcCfg<BN, X3>;
  static std::atomic<unsigned long long> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaError_t e =
        cudaFuncSetAttribute(tc_conv_kernel<BN, X3>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return e;
  }
  long long tiles = tc_conv_max_tiles(p, BN);
  if (p.mode == 0 && p.ks_max > 1) tiles *= p.ks_max;
  if (tiles <= 0) return cudaSuccess;
  const int grid = tiles < num_sms ? static_cast<int>(tiles) : num_sms;
  return launch_pdl(tc_conv_kernel<BN, X3>, dim3(grid), dim3(kThreads), Cfg::kSmem, stream, p);
}

}  // namespace

bool encode_act_map(CUtensorMap* map, const void* base, int C, int W, int H, int N, int P, int wb, int hb, int stride,
                    int nbox) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(P)};
  cuuint64_t strides[4];
  strides[0] = static_cast<cuuint64_t>(C) * 2;
  strides[1] = strides[0] * W;
  strides[2] = strides[1] * H;
  strides[3] = strides[2] * N;
  const cuuint32_t st = static_cast<cuuint32_t>(stride < 1 ? 1 : stride);
  // With traversal stride st, TMA loads boxDim/st elements: box = wanted * st.
  cuuint32_t box[5] = {64, static_cast<cuuint32_t>(wb) * st, static_cast<cuuint32_t>(hb) * st,
                       static_cast<cuuint32_t>(nbox < 1 ? 1 : nbox), 1};
  cuuint32_t estr[5] = {1, st, st, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_weight_map(CUtensorMap* map, const void* base, int K, int Cout, int BN) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Cout)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BN)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int tc_conv_ring_bytes(int BN, bool x3) {
  switch (BN) {
    case 64:
      return x3 ? TcCfg<64, true>::kStages * TcCfg<64, true>::kStageBytes
                : TcCfg<64, false>::kStages * TcCfg<64, false>::kStageBytes;
    case 128:
      return x3 ? TcCfg<128, true>::kStages * TcCfg<128, true>::kStageBytes
                : TcCfg<128, false>::kStages * TcCfg<128, false>::kStageBytes;
    case 256:
      return x3 ? 0 : TcCfg<256, false>::kStages * TcCfg<256, false>::kStageBytes;
    default:
      return 0;
  }
}

bool tc_conv_halo_plan(int H, int W, int k, int stride, int pad, int Cout, bool x3, int& BN, HaloPlan& hp) {
  if (stride != 1 || k < 2 || pad != k / 2 || (k % 2) == 0) return false;
  const int Pw = W + 2 * pad;
  if (Pw < 16 || Pw > 256) return false;
  const int rows = (Pw - 1 + 127 + (k - 1) * (Pw + 1)) / Pw + 1;
  if (rows > 256) return false;
  const int planes = x3 ? 2 : 1;
  hp.pw = Pw;
  hp.rows = rows;
  hp.res_rows = (Pw - 1 + 127) / Pw + 1;
  hp.aplane = static_cast<unsigned>((Pw * rows * 128 + 1023) / 1024 * 1024);
  hp.tiles_per_img = (H * Pw + 127) / 128;
  for (int bn : {BN, 64}) {
    if (Cout % bn) continue;
    const long long ring = tc_conv_ring_bytes(bn, x3);
    const long long left = ring - 2LL * planes * hp.aplane;
    const int sb = left > 0 ? static_cast<int>(left / (static_cast<long long>(planes) * bn * 128)) : 0;
    if (sb >= 3) {
      BN = bn;
      hp.sb = sb > 8 ? 8 : sb;
      return true;
    }
  }
  return false;
}

int tc_conv_pick_bn(int Cout, int segs) {
  if (segs == 1 && Cout % 256 == 0 && Cout >= 512) return 256;
  if (Cout % 128 == 0) return 128;
  return 64;
}

int tc_conv_max_tiles(const TcConvParams& p, int BN) {
  const int count = p.count_static;
  long long n_groups, tiles_w;
  if (p.plain) {
    n_groups = 1;
    tiles_w = (count + kBM - 1) / kBM;
  } else {
    n_groups = (count + p.ipt - 1) / p.ipt;
    tiles_w = p.tiles_w;
  }
  const long long total = n_groups * p.tiles_h * tiles_w * (p.Cout / BN) * (p.mode == 1 ? p.ksplit : 1);
  return total > 0x7fffffff ? 0x7fffffff : static_cast<int>(total);
}

size_t tc_conv_ws_floats(int BN, int max_ctas) { return 2ull * static_cast<size_t>(max_ctas) * kBM * BN; }

cudaError_t tc_conv_launch(const TcConvParams& p, int BN, int num_sms, cudaStream_t stream) {
  const bool x3 = p.segs == 3;
  if (p.res_proj && (p.halo || p.nres <= 0)) return cudaErrorInvalidValue;  // the halo producer has no projection path
  switch (BN) {
    case 64:
      return x3 ? launch_cfg<64, true>(p, num_sms, stream) : launch_cfg<64, false>(p, num_sms, stream);
    case 128:
      return x3 ? launch_cfg<128, true>(p, num_sms, stream) : launch_cfg<128, false>(p, num_sms, stream);
    case 256:
      return x3 ? cudaErrorInvalidValue : launch_cfg<256, false>(p, num_sms, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace lcb
