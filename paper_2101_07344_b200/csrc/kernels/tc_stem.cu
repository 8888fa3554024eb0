// tcgen05 stem convolution over the space-to-depth image X (see tc_stem.cuh).
//
// Warp roles (one persistent CTA per SM; 2 + 8 * SETS warps):
//   warp 0     : producer (lane 0): resident weights once, then one X slab per
//                tile (bulk copies, 2 groups x planes) into a ring of stages
//   warp 1     : MMA issuer (whole warp, elect.sync): k'^2 taps x {1, 2} MMAs (M128, N 64 / stacked 128, K16)
//   warps 2..  : epilogue (TMEM lane quadrant warp % 4, column half ((warp-2)/4) % 2): folded BN, ReLU,
//                hi/lo split, NHWC store of the valid anchors. SETS = 2: two sets of
//                8 warps, set s drains TMEM accumulator s (the CTA's tiles 2i + s), so
//                one set's dependent chain (TMEM load -> exchange barrier -> shuffles
//                -> stores) overlaps the other's — with one set the epilogue's
//                latency, not the tensor pipe (44 % busy), set the stem's tile rate
#include <cfloat>
#include <cstdlib>
#include <type_traits>

#include "pdl.cuh"
#include "sm100_prims.cuh"
#include "tc_stem.cuh"

namespace lcb {

namespace {

constexpr int kBM = 128;
constexpr int kCout = 64;
constexpr int kTapBytes = 2 * kCout * 16;  // [2 groups][64 rows][16 B]

__device__ __forceinline__ float4 u4_as_f4(uint4 u) {
  return make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w));
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
               : "memory");
}

// No-swizzle K-major descriptor: core matrix = 8 rows x 16 B (rows 16 B
// apart); lbo = byte distance between the two K-adjacent core matrices
// (channel groups), sbo = byte distance between 8-row groups (128 B).
__device__ __forceinline__ uint64_t desc_kmajor_none(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(128 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // sm_100 descriptor version; layout type 0 = no swizzle
  return d;
}

struct StemSmem {
  int planes, taps, npix_alloc, stages;
  uint32_t w_bytes, stage_bytes, group_bytes, plane_bytes, epi_bytes;
};

// epilogue scratch: 4 KB store staging per epilogue warp (direct stores), or
// the hpool path's left-neighbour exchange (4 buffers x 2 halves x 4 quads x 32 floats)
__host__ __device__ inline StemSmem stem_smem(int x3, int kk, int Wx, int hpool, int sets) {
  StemSmem s;
  s.planes = x3 ? 2 : 1;
  s.taps = kk * kk;
  const int npix = kBM + (kk - 1) * (Wx + 1);
  s.npix_alloc = (npix + 7) / 8 * 8;
  s.group_bytes = static_cast<uint32_t>(s.npix_alloc) * 16;
  s.plane_bytes = 2 * s.group_bytes;
  s.stage_bytes = s.planes * s.plane_bytes;
  s.w_bytes = static_cast<uint32_t>(s.planes * s.taps * kTapBytes);
  s.epi_bytes = hpool ? 4096u : static_cast<uint32_t>(sets) * 8u * 4096u;
  int st = static_cast<int>((220u * 1024u - 2u * 1024u - s.epi_bytes - s.w_bytes) / s.stage_bytes);
  s.stages = st > 8 ? 8 : st;
  return s;
}

// KK > 0: compile-time taps per dimension (the MMA issue loop fully unrolled); 0: p.kk.
template <bool X3, int KK, int SETS>
__global__ void __launch_bounds__(64 + 256 * SETS, 1) tc_stem_kernel(const __grid_constant__ StemParams p) {
  const int kk = KK > 0 ? KK : p.kk;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const StemSmem L = stem_smem(X3 ? 1 : 0, kk, p.Wx, p.hpool, SETS);
  const int S = L.stages;
  uint8_t* wsm = smem;
  uint8_t* slabs = smem + L.w_bytes;
  uint8_t* epi = slabs + S * L.stage_bytes;  // epilogue scratch, then 64 floats of shift
  float* shift_s = reinterpret_cast<float*>(epi + L.epi_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + L.epi_bytes + 256);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * 8 + 5);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = smem_u32(bars + 8);
  const uint32_t tfull0 = smem_u32(bars + 16);
  const uint32_t tempty0 = smem_u32(bars + 18);
  const uint32_t wbar = smem_u32(bars + 20);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull0 + 8 * i, 1);
      mbar_init(tempty0 + 8 * i, 8);
    }
    mbar_init(wbar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < kCout) shift_s[threadIdx.x] = p.shift[threadIdx.x];
  // bf16x3: accumulators are [hi*hi | hi*lo] = 2 x 64 columns (the stacked MMA below)
  constexpr uint32_t kAccCols = X3 ? 2 * kCout : kCout;
  if (warp == 0) tmem_alloc(smem_u32(tmem_holder), 2 * kAccCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();  // programmatic launch: the prologue above overlaps the previous kernel
  pdl_trigger();

  const int count = *p.count;
  const int total = count * p.tiles_per_img;
  const int HWx = p.Hx * p.Wx;
  const int npix = kBM + (kk - 1) * (p.Wx + 1);

  if (warp == 0) {
    {
      // ------------------------------------------------ producer (whole warp:
      // the planes x groups bulk copies of a slab go out from separate lanes)
      if (lane == 0) {  // resident weights (bf16x3: one stacked [tap][group][hi 64 | lo 64][8] buffer)
        mbar_expect_tx(wbar, L.w_bytes);
        bulk_g2s(smem_u32(wsm), p.w_hi, L.w_bytes, wbar);
      }
      const int pl = lane >> 1, grp = lane & 1;  // lane's copy: plane, channel group
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int n = t / p.tiles_per_img;
        const int m0 = (t - n * p.tiles_per_img) * (p.hpool ? p.Wx : kBM);  // hpool: one output row per tile
        const int len = npix < HWx - m0 ? npix : HWx - m0;
        mbar_wait(empty0 + 8 * stage, phase ^ 1);
        const uint32_t fb = full0 + 8 * stage;
        if (lane == 0) mbar_expect_tx(fb, static_cast<uint32_t>(L.planes * 2 * len * 16));
        __syncwarp();
        if (pl < L.planes) {
          uint8_t* st = slabs + stage * L.stage_bytes;
          const __nv_bfloat16* xp = pl == 0 ? p.x_hi : p.x_lo;
          const __nv_bfloat16* src = xp + ((static_cast<size_t>(n) * 2 + grp) * HWx + m0) * 8;
          bulk_g2s(smem_u32(st + pl * L.plane_bytes + grp * L.group_bytes), src, static_cast<uint32_t>(len * 16), fb);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp, warp-uniform operands, elect.sync issues (a single-lane
       // loop capped the issue rate near one MMA per 130 cycles, sm100_prims.cuh)
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, kCout);
      constexpr uint32_t idesc2 = umma_idesc_bf16(kBM, 2 * kCout);  // stacked [B_hi; B_lo]
      mbar_wait(wbar, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        mbar_wait(full0 + 8 * stage, phase);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        const uint32_t a0 = smem_u32(slabs + stage * L.stage_bytes);
        const uint32_t b0 = smem_u32(wsm);
        // descriptors built once per tile; a tap moves the start address field
        // (bits 0-13, 16-byte units) by its row shift / weight offset
        const uint64_t da_hi = desc_kmajor_none(a0, L.group_bytes);
        const uint64_t da_lo = desc_kmajor_none(a0 + L.plane_bytes, L.group_bytes);
        // bf16x3 weights per tap: [group][hi 64 rows | lo 64 rows][8] (LBO =
        // 2 KB between the channel groups): hi*[W_hi; W_lo] is ONE N = 128 MMA
        // into [cols 0, 64) | [64, 128), then lo*W_hi (the first 64 rows) into
        // the low half — 2 MMAs per tap instead of 3; the epilogue adds the halves
        const uint64_t db = desc_kmajor_none(b0, (X3 ? 2 : 1) * kCout * 16);
        constexpr uint64_t kTapStep = (X3 ? 2 : 1) * kTapBytes / 16;
        uint32_t accum = 0;
        uint64_t bo = 0;
#pragma unroll
        for (int r = 0; r < (KK > 0 ? KK : kk); ++r) {
          uint64_t ao = static_cast<uint64_t>(r * p.Wx);
#pragma unroll
          for (int s = 0; s < (KK > 0 ? KK : kk); ++s, ++ao, bo += kTapStep) {
            if (X3) {
              umma_bf16_warp(d_tmem, da_hi + ao, db + bo, idesc2, accum);
              umma_bf16_warp(d_tmem, da_lo + ao, db + bo, idesc, 1u);
            } else {
              umma_bf16_warp(d_tmem, da_hi + ao, db + bo, idesc, accum);
            }
            accum = 1u;
          }
        }
        umma_commit_warp(empty0 + 8 * stage);
        umma_commit_warp(tfull0 + 8 * acc);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------ epilogue (8 warps per set: TMEM lane quadrant
    // warp % 4, column half ((warp - 2) / 4) % 2; set (warp - 2) / 8 drains accumulator `set`
    // when SETS = 2, both accumulators in turn when SETS = 1)
    const int quad = warp & 3;
    const int q = ((warp - 2) >> 2) & 1;
    const int set = (warp - 2) >> 3;
    const int row = quad * 32 + lane;
    int acc = SETS == 2 ? set : 0;
    uint32_t acc_phase = 0;
    int iter = 0;
    const int HoWx = p.Ho * p.Wx;
    for (int t = blockIdx.x + set * gridDim.x; t < total; t += SETS * gridDim.x, ++iter) {
      const int n = t / p.tiles_per_img;
      const int m = (t - n * p.tiles_per_img) * (p.hpool ? p.Wx : kBM) + row;
      const int oh = p.hpool ? t - n * p.tiles_per_img : m / p.Wx;
      const int ow = p.hpool ? row : m - (m / p.Wx) * p.Wx;
      const bool valid = m < HoWx && ow < p.Wo;
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * kAccCols;
      float v[2][16];
#pragma unroll
      for (int c = 0; c < 2; ++c) tmem_ld16_nowait(t_row + q * 32 + c * 16, v[c]);
      if (X3) {  // + the hi*lo half
        float w[2][16];
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_ld16_nowait(t_row + kCout + q * 32 + c * 16, w[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 16; ++e) v[c][e] += w[c][e];
      } else {
        tmem_ld_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
      // exchange buffer: alternates between consecutive tiles of the same warps
      // (a fast warp's next write must not land on a slow warp's pending read)
      const int xbuf = SETS == 2 ? set * 2 + (iter & 1) : acc;
      if (SETS == 2) {
        acc_phase ^= 1;
      } else {
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      if (p.hpool) {
        // folded BN shift + ReLU in fp32; anchors past the row are -inf for the max
        // (shared operands through explicit 16-byte ld.shared: the aligned smem
        // base is an integer round trip, so plain pointers compile to generic
        // loads, and the MIO queue — shared by 16 epilogue warps' shuffles — is
        // the epilogue's throttle)
        float a[32];
        const uint32_t sh_addr = smem_u32(shift_s + q * 32);
#pragma unroll
        for (int u4 = 0; u4 < 8; ++u4) {
          const float4 s4 = u4_as_f4(ld_shared_v4(sh_addr + u4 * 16));
          const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = u4 * 4 + k;
            float z = v[i >> 4][i & 15] + sv[k];
            if (p.relu) z = z > 0.0f ? z : 0.0f;
            a[i] = valid ? z : -FLT_MAX;
          }
        }
        // left neighbour (ow - 1): the lane below, or lane 31 of the previous
        // quad's warp through shared memory (double-buffered by accumulator)
        float* xch = reinterpret_cast<float*>(epi) + ((xbuf * 2 + q) * 4) * 32;  // [quad][32 channels]
        if (lane == 31)
#pragma unroll
          for (int c = 0; c < 32; c += 4)
            *reinterpret_cast<float4*>(xch + quad * 32 + c) = make_float4(a[c], a[c + 1], a[c + 2], a[c + 3]);
        asm volatile("bar.sync %0, 128;" ::"r"(2 + 2 * set + q) : "memory");  // the four quads of this column half
        // lane 0's left neighbours: lane 31 of the previous row block (quad - 1)
        const uint32_t lx_addr = smem_u32(xch + ((quad + 3) & 3) * 32);
        // lane pairs (ow, ow + 1), ow even, share the pooled pixel ow: the even lane
        // writes its channels [0, 16), the odd lane [16, 32) — 48 shuffles per lane
        // instead of 64 (one exchange inside the pair, the left neighbour's two halves)
        const int odd = lane & 1;
        const int pw = ow - odd;  // the pooled anchor (even)
        const int src_l = (odd ? lane - 2 : lane - 1) & 31;
        uint4 hi[2], lo[2];
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(hi);
        __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(lo);
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          float lv[2] = {-FLT_MAX, -FLT_MAX};
          if (lane < 2 && quad != 0) {  // lane 31 of the previous row block, this lane's half
            uint32_t x0, x1;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x0), "=r"(x1) : "r"(lx_addr + (odd * 16 + k) * 4));
            lv[0] = __uint_as_float(x0);
            lv[1] = __uint_as_float(x1);
          }
          float mx[2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const int c = k + d;
            const float mine = odd ? a[16 + c] : a[c];
            // even lane: a[ow + 1][c]; odd lane: a[ow - 1][16 + c]
            const float pair = __shfl_xor_sync(0xffffffffu, odd ? a[c] : a[16 + c], 1);
            const float l0 = __shfl_sync(0xffffffffu, a[c], src_l);
            const float l1 = __shfl_sync(0xffffffffu, a[16 + c], src_l);
            const float left = lane < 2 ? lv[d] : (odd ? l1 : l0);
            // first maximum in (pw - 1, pw, pw + 1) order
            const float mid = odd ? pair : mine, right = odd ? mine : pair;
            float m = left;
            if (mid > m) m = mid;
            if (right > m) m = right;
            mx[d] = m;
          }
          const __nv_bfloat162 hh = __floats2bfloat162_rn(mx[0], mx[1]);
          h2[k / 2] = hh;
          const float2 hf = __bfloat1622float2(hh);
          l2[k / 2] = __floats2bfloat162_rn(mx[0] - hf.x, mx[1] - hf.y);
        }
        if (pw < p.Wo && m - odd < HoWx) {
          const size_t ob = ((static_cast<size_t>(n) * p.Ho + oh) * p.Wp + (pw >> 1)) * kCout + q * 32 + odd * 16;
          uint4* oh4 = reinterpret_cast<uint4*>(p.out_hi + ob);
          oh4[0] = hi[0];
          oh4[1] = hi[1];
          if (X3 && p.out_lo) {
            uint4* ol4 = reinterpret_cast<uint4*>(p.out_lo + ob);
            ol4[0] = lo[0];
            ol4[1] = lo[1];
          }
        }
        continue;
      }
      // staged, coalesced stores: 32 rows x 32 channels per step, 8 rows x 64 B per instruction
      const unsigned long long off = valid ? ((static_cast<unsigned long long>(n) * p.Ho + oh) * p.Wo + ow) * kCout : 0ull;
      const uint32_t wst = smem_u32(epi + (warp - 2) * 4096);
      {
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int cb = q * 32 + u * 16;
          uint4 hi[2], lo[2];
          __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(hi);
          __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(lo);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float a = v[u][2 * e] + shift_s[cb + 2 * e];
            float b = v[u][2 * e + 1] + shift_s[cb + 2 * e + 1];
            if (p.relu) {
              a = a > 0.0f ? a : 0.0f;
              b = b > 0.0f ? b : 0.0f;
            }
            const __nv_bfloat162 hh = __floats2bfloat162_rn(a, b);
            h2[e] = hh;
            const float2 hf = __bfloat1622float2(hh);
            l2[e] = __floats2bfloat162_rn(a - hf.x, b - hf.y);
          }
#pragma unroll
          for (int hq = 0; hq < 2; ++hq) {
            const uint32_t so = static_cast<uint32_t>(lane * 64 + (((u * 2 + hq) ^ ((lane >> 1) & 3)) * 16));
            st_shared_v4(wst + so, hi[hq]);
            if (X3) st_shared_v4(wst + 2048 + so, lo[hq]);
          }
        }
        __syncwarp();
        const int ch = lane & 3;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = (lane >> 2) + 8 * i;
          const unsigned long long ob = __shfl_sync(0xffffffffu, off, r);
          const int ok = __shfl_sync(0xffffffffu, valid ? 1 : 0, r);
          const uint32_t so = static_cast<uint32_t>(r * 64 + ((ch ^ ((r >> 1) & 3)) * 16));
          if (ok) {
            *reinterpret_cast<uint4*>(p.out_hi + ob + q * 32 + ch * 8) = ld_shared_v4(wst + so);
            if (X3 && p.out_lo) *reinterpret_cast<uint4*>(p.out_lo + ob + q * 32 + ch * 8) = ld_shared_v4(wst + 2048 + so);
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tmem_dealloc(tmem_base, 2 * kAccCols);
  }
}

// One thread per (image, channel group, X pixel): 8 channels -> 16-byte stores.
__global__ void stem_s2d_kernel(const float* x, const int* count, int C, int H, int W, int stride, int pad, int Hx,
                                int Wx, __nv_bfloat16* x_hi, __nv_bfloat16* x_lo) {
  pdl_wait();
  pdl_trigger();
  // 32-bit index math (the batch's X has < 2^31 units): 64-bit divisions per
  // element made this kernel ALU-bound
  const unsigned HWx = static_cast<unsigned>(Hx) * Wx;
  const unsigned total = static_cast<unsigned>(*count) * 2u * HWx;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned ng = i / HWx, pix = i - ng * HWx;  // ng = n * 2 + grp
    const int grp = static_cast<int>(ng & 1u);
    const long long n = ng >> 1;
    const int I = static_cast<int>(pix / static_cast<unsigned>(Wx)), J = static_cast<int>(pix - I * static_cast<unsigned>(Wx));
    const float* xn = x + n * C * H * W;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int q = grp * 8 + e;
      int c, ih, iw;
      if (stride == 2) {
        c = q >> 2;
        ih = 2 * I + ((q >> 1) & 1) - pad;
        iw = 2 * J + (q & 1) - pad;
      } else {
        c = q;
        ih = I - pad;
        iw = J - pad;
      }
      v[e] = (c < C && ih >= 0 && ih < H && iw >= 0 && iw < W) ? xn[(static_cast<long long>(c) * H + ih) * W + iw]
                                                               : 0.0f;
    }
    uint4 h4, l4;
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&h4);
    __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&l4);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      h2[e] = hh;
      const float2 hf = __bfloat1622float2(hh);
      l2[e] = __floats2bfloat162_rn(v[2 * e] - hf.x, v[2 * e + 1] - hf.y);
    }
    reinterpret_cast<uint4*>(x_hi)[i] = h4;
    if (x_lo) reinterpret_cast<uint4*>(x_lo)[i] = l4;
  }
}

// Vertical 3-row max (stride 2, pad 1) over the hpool stem output, one thread
// per (image, pooled pixel, 8 channels), 16-byte loads; hi and lo move together.
__global__ void stem_vpool_kernel(const __nv_bfloat16* in_hi, const __nv_bfloat16* in_lo, int Hi, int Wp, int C,
                                  int Hp, const int* ids, const int* count, __nv_bfloat16* out_hi,
                                  __nv_bfloat16* out_lo) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x;
  if (j >= *count) return;
  const long long n = ids ? ids[j] : j;
  const int c8n = C / 8;
  const int per = Hp * Wp * c8n;  // (32-bit index math per element)
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < per; i += gridDim.y * blockDim.x) {
    const int pix = i / c8n, c8 = i - pix * c8n;
    const int pi = pix / Wp, pj = pix - pi * Wp;
    uint4 vh[3], vl[3];
    bool ok[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int ir = 2 * pi - 1 + r;
      ok[r] = ir >= 0 && ir < Hi;
      const long long src = ((n * Hi + (ok[r] ? ir : 0)) * Wp + pj) * C + c8 * 8;
      vh[r] = ok[r] ? __ldg(reinterpret_cast<const uint4*>(in_hi + src)) : make_uint4(0, 0, 0, 0);
      vl[r] = ok[r] && in_lo ? __ldg(reinterpret_cast<const uint4*>(in_lo + src)) : make_uint4(0, 0, 0, 0);
    }
    float best[8];
    uint4 bh = make_uint4(0, 0, 0, 0), bl = make_uint4(0, 0, 0, 0);
    __nv_bfloat16* bh8 = reinterpret_cast<__nv_bfloat16*>(&bh);
    __nv_bfloat16* bl8 = reinterpret_cast<__nv_bfloat16*>(&bl);
#pragma unroll
    for (int e = 0; e < 8; ++e) best[e] = -FLT_MAX;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      if (!ok[r]) continue;
      const __nv_bfloat16* h8 = reinterpret_cast<const __nv_bfloat16*>(&vh[r]);
      const __nv_bfloat16* l8 = reinterpret_cast<const __nv_bfloat16*>(&vl[r]);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v = __bfloat162float(h8[e]) + __bfloat162float(l8[e]);
        if (v > best[e]) {
          best[e] = v;
          bh8[e] = h8[e];
          bl8[e] = l8[e];
        }
      }
    }
    const long long dst = ((n * Hp + pi) * Wp + pj) * C + c8 * 8;
    *reinterpret_cast<uint4*>(out_hi + dst) = bh;
    if (out_lo) *reinterpret_cast<uint4*>(out_lo + dst) = bl;
  }
}

}  // namespace

void launch_stem_vpool(const __nv_bfloat16* in_hi, const __nv_bfloat16* in_lo, int Hi, int Wp, int C, int Hp,
                       const int* ids, const int* count, int max_rows, __nv_bfloat16* out_hi, __nv_bfloat16* out_lo,
                       cudaStream_t s) {
  if (max_rows <= 0) return;
  const long long per = static_cast<long long>(Hp) * Wp * (C / 8);
  int gy = static_cast<int>((per + 255) / 256);
  if (gy > 128) gy = 128;
  launch_pdl(stem_vpool_kernel, dim3(max_rows, gy), dim3(256), 0, s, in_hi, in_lo, Hi, Wp, C, Hp, ids, count, out_hi,
             out_lo);
}

StemGeom stem_geom(int H, int W, int k, int stride, int pad) {
  StemGeom g;
  g.Ho = (H + 2 * pad - k) / stride + 1;
  g.Wo = (W + 2 * pad - k) / stride + 1;
  if (stride == 2) {
    g.kk = (k + 1) / 2;
    g.Hx = g.Ho + g.kk - 1;
    g.Wx = g.Wo + g.kk - 1;
  } else {
    g.kk = k;
    g.Hx = H + 2 * pad;
    g.Wx = W + 2 * pad;
  }
  return g;
}

void stem_weights(const double* w, int Cout, int C, int k, int stride, const StemGeom& g, float* out) {
  // out[tap][grp][o][e], channel q = grp*8 + e of X
  for (int tr = 0; tr < g.kk; ++tr)
    for (int ts = 0; ts < g.kk; ++ts)
      for (int grp = 0; grp < 2; ++grp)
        for (int o = 0; o < Cout; ++o)
          for (int e = 0; e < 8; ++e) {
            const int q = grp * 8 + e;
            int c, r, s;
            if (stride == 2) {
              c = q >> 2;
              r = 2 * tr + ((q >> 1) & 1);
              s = 2 * ts + (q & 1);
            } else {
              c = q;
              r = tr;
              s = ts;
            }
            double v = 0.0;
            if (c < C && r < k && s < k) v = w[((static_cast<size_t>(o) * C + c) * k + r) * k + s];
            out[(((static_cast<size_t>(tr) * g.kk + ts) * 2 + grp) * Cout + o) * 8 + e] = static_cast<float>(v);
          }
}

void launch_stem_s2d(const float* x, const int* count, int max_n, int C, int H, int W, int stride, int pad,
                     const StemGeom& g, __nv_bfloat16* x_hi, __nv_bfloat16* x_lo, cudaStream_t s) {
  const long long total = static_cast<long long>(max_n) * 2 * g.Hx * g.Wx;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  launch_pdl(stem_s2d_kernel, dim3(static_cast<int>(blocks)), dim3(256), 0, s, x, count, C, H, W, stride, pad, g.Hx, g.Wx, x_hi, x_lo);
}

cudaError_t tc_stem_launch(const StemParams& p, int num_sms, cudaStream_t stream) {
  const bool x3 = p.x_lo != nullptr;
  if (p.hpool && (p.Wx > kBM || p.tiles_per_img != p.Ho || p.Wp != (p.Wo - 1) / 2 + 1)) return cudaErrorInvalidValue;
  // LCB_STEM_EPI_SETS=1: one set of 8 epilogue warps (the round-2 layout, kept for A/B)
  static const int sets = [] {
    const char* e = std::getenv("LCB_STEM_EPI_SETS");
    return e && std::atoi(e) == 1 ? 1 : 2;
  }();
  const StemSmem L = stem_smem(x3 ? 1 : 0, p.kk, p.Wx, p.hpool, sets);
  if (L.stages < 2) return cudaErrorInvalidValue;
  const size_t smem = L.w_bytes + static_cast<size_t>(L.stages) * L.stage_bytes + L.epi_bytes + 256 + 256 + 1024;
  const long long tiles = static_cast<long long>(p.count_static) * p.tiles_per_img;
  if (tiles <= 0) return cudaSuccess;
  const int grid = tiles < num_sms ? static_cast<int>(tiles) : num_sms;
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    launch_pdl(kern, dim3(grid), dim3(64 + 256 * sets), smem, stream, p);
    return cudaGetLastError();
  };
  auto pick = [&](auto x3c, auto setsc) {
    constexpr bool X = decltype(x3c)::value;
    constexpr int E = decltype(setsc)::value;
    return p.kk == 4 ? go(tc_stem_kernel<X, 4, E>) : p.kk == 3 ? go(tc_stem_kernel<X, 3, E>) : go(tc_stem_kernel<X, 0, E>);
  };
  using T = std::true_type;
  using F = std::false_type;
  using One = std::integral_constant<int, 1>;
  using Two = std::integral_constant<int, 2>;
  if (x3) return sets == 2 ? pick(T{}, Two{}) : pick(T{}, One{});
  return sets == 2 ? pick(F{}, Two{}) : pick(F{}, One{});
}

}  // namespace lcb
