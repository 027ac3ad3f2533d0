// spectral_fused.cuh — the row and column passes of a spectral step in ONE
// persistent, warp-specialised kernel (included by spectral.cu inside its
// anonymous namespace; N = 1024). OPT-IN (OCN_FUSED=1): slower than the
// two-kernel step on B200, see fused_enabled() in spectral.cu for the numbers.
//
// Why: the two-kernel step round-trips every transform's row-pass result
// through HBM (16 B / point / transform, ~2x the compulsory bytes of the
// path), and the issue-bound row pass and the HBM-bound column pass run one
// after the other. Here each SM runs both at once:
//   * 8 row warps take row tasks (wave w, row i) from a global counter: stage
//     the grid's row of (h~, G)-derived coefficients, each warp transforms one
//     of the wave's <= 8 transforms and writes scratch slot w % kFuseSlots;
//   * 4 column warps take column tiles (wave w, transform, 4 columns) from a
//     second counter, fed by a 3-stage TMA ring (cp.async.bulk.tensor +
//     mbarrier) exactly like k_cols_tma, and write the output fields.
// Waves are <= kFuseW transforms of one grid and family; only kFuseSlots waves
// of scratch exist (128 MB at N = 1024), meant to keep the column tiles' reads
// in L2. Tasks are assigned statically (row task / tile k of a CTA = blockIdx.x
// + k gridDim.x, in order). Dependencies are per-wave counters in global memory:
//   column tile of wave w   waits  rows_done[w]  == N
//   row task of wave w      waits  tiles_done[w - kFuseSlots] == tiles(w - kFuseSlots)
// (release: a named barrier, then one thread's __threadfence + atomicAdd of
// the CTA's count when it leaves a wave; acquire: ld.acquire.gpu +
// fence.proxy.async before the TMA read). A group only blocks while it holds
// no unfinished task (a column tile whose wave is not ready is parked
// "pending" and waited for at the top of the loop) and every dependency points
// at an earlier wave, so with all CTAs resident (grid = SM count, one CTA per
// SM) the schedule cannot deadlock.
#pragma once

#ifndef OCN_FUSE_W
#define OCN_FUSE_W 8
#endif
#ifndef OCN_FUSE_SLOTS
#define OCN_FUSE_SLOTS 2
#endif
constexpr int kFuseW = OCN_FUSE_W;          // transforms per wave (<= one per row warp)
constexpr int kFuseSlots = OCN_FUSE_SLOTS;  // scratch slots = waves in flight
constexpr int kFuseRowWarps = 8;
constexpr int kFuseColWarps = 4;
constexpr int kFuseColStages = 3;
constexpr int kFusePending = 1 << 30;  // stage tile id flag: claimed, load not issued
constexpr int kFuseEnd = -1;           // stage: no more tiles

struct FusedWave {
  int grid, family, first, count;  // transforms [first, first + count) of the plan
};

struct FusedArgs {
  const float2* spec_h;  // h~ of every grid, [grid][N][N]
  const float2* spec_g;  // G of every grid
  const GridConst* gc;
  float chop;
  const XformDesc* desc;   // plan descriptors
  const FusedWave* waves;  // [nwaves]
  const int* tile0;        // column tiles before wave w, [nwaves + 1]
  int nwaves;
  float2* scratch;  // [kFuseSlots * kFuseW][N][N] (the first transforms of the cascade scratch)
  const float2* tw;
  int* ctr;  // [0] row tasks claimed, [1] tiles claimed, [2, 2 + nw) rows done, then tiles done
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
template <int ID, int COUNT>
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}

template <int N>
struct Fused {
  using PL = fft::Plan<N>;
  static_assert(PL::T == 32 && PL::P == 2, "the fused step is written for N = 1024");
  static constexpr int T = PL::T;
  static constexpr int ROW_THREADS = 32 * kFuseRowWarps;
  static constexpr int COL_THREADS = 32 * kFuseColWarps;
  static constexpr int THREADS = ROW_THREADS + COL_THREADS;
  static constexpr int PC = COL_THREADS / T;  // columns per tile
  static constexpr int CSTRIDE = fft::col_stride(PL::SMEM, PC);
  static constexpr int DENSE = N * PC;
  static constexpr int STAGE = ((DENSE > PC * CSTRIDE ? DENSE : PC * CSTRIDE) + 15) / 16 * 16;
  static constexpr int TILES_PER_XF = N / PC;
  static constexpr uint32_t TILE_BYTES = (uint32_t)DENSE * 8;
  static constexpr int RSTRIDE = PL::SMEM;
  // shared layout (float2 units): row staging (20 B / mode), twiddles, row
  // warp buffers, column stages, then ints and mbarriers
  static constexpr int STG = (5 * N / 2 + 15) / 16 * 16;
  static constexpr int TWN = (PL::tw_size() + 15) / 16 * 16;
  static constexpr int OFF_TW = STG;
  static constexpr int OFF_RB = OFF_TW + TWN;
  static constexpr int OFF_CS = OFF_RB + (kFuseRowWarps * RSTRIDE + 15) / 16 * 16;
  static constexpr int OFF_END = OFF_CS + kFuseColStages * STAGE;
  static constexpr size_t SMEM = (size_t)OFF_END * 8 + 32 * sizeof(int) + kFuseColStages * 8;
};

template <int N>
__global__ void __launch_bounds__(Fused<N>::THREADS, 1)
    k_spectral_fused(const __grid_constant__ CUtensorMap src, const FusedArgs a) {
  using F = Fused<N>;
  constexpr int H = N / 2;  // centring half-shift (kCentreByShift)
  extern __shared__ __align__(128) float2 smem[];
  float2* stw = smem + F::OFF_TW;
  int* sint = reinterpret_cast<int*>(smem + F::OFF_END);  // [0, 8): per stage; [8]: row task
  const uint32_t bar0 = tma::smem_u32(sint + 32);
  const int tid = threadIdx.x;
  for (int i = tid; i < F::PL::tw_size(); i += F::THREADS) stw[i] = __ldg(a.tw + i);
  if (tid == F::ROW_THREADS) {
    for (int s = 0; s < kFuseColStages; ++s) tma::mbar_init(bar0 + 8 * s, 1);
    tma::fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier: the roles below never meet again
  int* rows_done = a.ctr + 2;
  int* tiles_done = a.ctr + 2 + a.nwaves;
  const int total_rows = a.nwaves * N;

  if (tid < F::ROW_THREADS) {
    // ------------------------------------------------------------ row role
    const int warp = tid >> 5, t = tid & 31;
    float2* buf = smem + F::OFF_RB + warp * F::RSTRIDE;
    // staging: velocity sv0 [0, N), sw0 [N, 2N), sk (float) at 2N; surface
    // sht [0, N), sinv (float) at N
    float2* sv0 = smem;
    float2* sw0 = smem + N;
    float* sk = reinterpret_cast<float*>(smem + 2 * N);
    float2* sht = smem;
    float* sinv = reinterpret_cast<float*>(smem + N);
    int slot_ready = kFuseSlots - 1;  // waves <= this have their scratch slot free
    int mine = 0;                     // rows of the current wave done by this CTA
    for (int task = blockIdx.x; task < total_rows; task += gridDim.x) {
      const int w = task / N, row = task - w * N;
      if (w > slot_ready) {  // the slot's previous wave must be fully read
        if (tid == 0) {
          const int wp = w - kFuseSlots, need = a.tile0[wp + 1] - a.tile0[wp];
          while (ld_acquire(tiles_done + wp) < need) __nanosleep(256);
        }
        slot_ready = w;
        named_sync<1, F::ROW_THREADS>();
      }
      const FusedWave wv = a.waves[w];
      const GridConst& gcv = a.gc[wv.grid];
      const float dk = (float)gcv.dk, g = (float)gcv.p.gravity;
      const float kx = dk * (float)(row - N / 2);
      const float2* srow = (wv.family == 0 ? a.spec_h : a.spec_g) + ((size_t)wv.grid * N + row) * N;
#pragma unroll 4
      for (int j = tid; j < N; j += F::ROW_THREADS) {
        const float2 sp = __ldg(srow + j);  // h~ (surface) or G (velocity)
        const float kz = dk * (float)(j - N / 2);
        const float k2 = kx * kx + kz * kz;
        const bool zero = k2 == 0.f;
        const float inv = zero ? 0.f : rsqrtf(k2);
        const float k = k2 * inv;
        if (wv.family == 0) {
          sht[j] = sp;
          sinv[j] = inv;
        } else {
          const float rw = zero ? 0.f : rsqrtf(g * k);
          const float wq = g * k * rw, f = -g * rw;
          sv0[j] = make_float2(f * (sp.x * kx - sp.y * kz), f * (sp.x * kz + sp.y * kx));
          sw0[j] = make_float2(sp.x * wq, sp.y * wq);
          sk[j] = k;
        }
      }
      named_sync<1, F::ROW_THREADS>();
      for (int xi = warp; xi < wv.count; xi += kFuseRowWarps) {
        const XformDesc d = a.desc[wv.first + xi];
        float2* out =
            a.scratch + ((size_t)((w % kFuseSlots) * kFuseW + xi) * N + (row ^ H)) * N;
        auto store = [&](int k, float2 x) { out[k] = x; };
        if (wv.family == 0) {
          // surface pairs (see k_rows_w): one branch-free form
          const float chop = a.chop;
          float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, c5 = 0.f, c6 = 0.f;
          if (d.kind == kSurfHDx) c0 = 1.f, c1 = -chop;
          else if (d.kind == kSurfDzDxDx) c5 = chop;
          else if (d.kind == kSurfDzDxDzDz) c2 = chop, c6 = chop;
          else c3 = -1.f, c4 = kx;
          const float kx2 = kx * kx;
          fft::cta_fft<N, true, false, false, true>(
              t, buf, stw,
              [&](int j) {
                const int jj = j ^ H;
                const float2 h = sht[jj];
                const float inv = sinv[jj];
                const float kz = dk * (float)(jj - N / 2);
                const float mr = fmaf(inv * kx, fmaf(c2, kz, c1), fmaf(c3, kz, c0));
                const float mi = fmaf(inv, fmaf(c6 * kz, kz, c5 * (kz + kx2)), c4);
                return make_float2(h.x * mr - h.y * mi, h.x * mi + h.y * mr);
              },
              store);
        } else {
          const float2* Z = d.kind == kVelXZ ? sv0 : sw0;
          constexpr float kLog2e = 1.4426950408889634f;
          const float y0 = d.y0, y1 = d.y1, y0l = y0 * kLog2e, y1l = y1 * kLog2e;
          const bool up0 = y0 > 0.f, up1 = y1 > 0.f;
          auto run = [&](auto kind_c) {
            constexpr int KIND = decltype(kind_c)::value;
            fft::cta_fft<N, true, false, false, true>(
                t, buf, stw,
                [&](int j) {
                  const int jj = j ^ H;
                  const float2 z = Z[jj];
                  const float k = sk[jj];
                  const float l0 = fmaf(k, y0, 1.0f), x0 = ex2_approx(k * y0l);
                  const float e0 = up0 ? l0 : x0;
                  if constexpr (KIND == kVelXZ) {
                    return make_float2(z.x * e0, z.y * e0);
                  } else if constexpr (KIND == kVelYPair) {
                    const float l1 = fmaf(k, y1, 1.0f), x1 = ex2_approx(k * y1l);
                    const float mr = -(up1 ? l1 : x1), mi = e0;
                    return make_float2(z.x * mr - z.y * mi, z.x * mi + z.y * mr);
                  } else {
                    return make_float2(-z.y * e0, z.x * e0);
                  }
                },
                store);
          };
          switch (d.kind) {
            case kVelXZ: run(std::integral_constant<int, kVelXZ>{}); break;
            case kVelYPair: run(std::integral_constant<int, kVelYPair>{}); break;
            default: run(std::integral_constant<int, kVelYSingle>{}); break;
          }
        }
      }
      named_sync<1, F::ROW_THREADS>();
      ++mine;
      const int next = task + gridDim.x;
      if (next >= total_rows || next / N != w) {  // this CTA's last row of wave w
        if (tid == 0) {  // release (cumulative over the barrier): the rows' scratch stores
          __threadfence();
          atomicAdd(rows_done + w, mine);
        }
        mine = 0;
      }
    }
  } else {
    // --------------------------------------------------------- column role
    constexpr int PC = F::PC, S = kFuseColStages;
    const int ctid = tid - F::ROW_THREADS;
    const int c = ctid % PC, t = ctid / PC;
    const bool leader = ctid == 0;
    const int total_tiles = a.tile0[a.nwaves];
    int* st_tile = sint;       // [S] claimed tile id (| kFusePending) or kFuseEnd
    int* st_xf = sint + 4;     // [S] plan transform index of the staged tile
    int* st_col = sint + 12;   // [S] first column
    int* st_wave = sint + 16;  // [S] wave
    auto wave_of = [&](int tile) {
      int lo = 0, hi = a.nwaves - 1;  // last w with tile0[w] <= tile
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(a.tile0 + mid) <= tile) lo = mid;
        else hi = mid - 1;
      }
      return lo;
    };
    auto issue = [&](int tile, int s) {  // leader only; the wave's rows are done
      const int w = wave_of(tile);
      const int local = tile - __ldg(a.tile0 + w);
      const int xi = local / F::TILES_PER_XF, cb = local - xi * F::TILES_PER_XF;
      st_tile[s] = tile;
      st_xf[s] = __ldg(&a.waves[w].first) + xi;
      st_col[s] = cb * PC;
      st_wave[s] = w;
      fence_proxy_async_global();
      tma::fence_proxy_async_smem();
      tma::mbar_arrive_expect_tx(bar0 + 8 * s, F::TILE_BYTES);
      tma::load_4d(tma::smem_u32(smem + F::OFF_CS + s * F::STAGE), &src, 2 * cb * PC, 0, 0,
                   (w % kFuseSlots) * kFuseW + xi, bar0 + 8 * s);
    };
    int next_tile = blockIdx.x;  // this CTA's tiles: blockIdx.x + k gridDim.x, in order
    int wave_ready = -1;         // leader: waves <= this have all rows done
    auto claim = [&](int s) {    // leader only, never blocks
      const int id = next_tile;
      next_tile += gridDim.x;
      if (id >= total_tiles) {
        st_tile[s] = kFuseEnd;
        return;
      }
      const int w = wave_of(id);
      if (w <= wave_ready || ld_acquire(rows_done + w) >= N) {
        wave_ready = w > wave_ready ? w : wave_ready;
        issue(id, s);
      } else {
        st_tile[s] = id | kFusePending;
      }
    };
    if (leader)
      for (int s = 0; s < S; ++s) claim(s);
    int s = 0, done_in_wave = 0;
    uint32_t phase = 0;
    for (;;) {
      if (leader) {
        const int v = st_tile[s];
        if (v != kFuseEnd && (v & kFusePending)) {  // holds no unfinished tile: may wait
          const int id = v & ~kFusePending;
          const int w = wave_of(id);
          while (ld_acquire(rows_done + w) < N) __nanosleep(128);
          wave_ready = w > wave_ready ? w : wave_ready;
          issue(id, s);
        }
      }
      named_sync<2, F::COL_THREADS>();
      if (st_tile[s] == kFuseEnd) break;
      const int xf = st_xf[s], col = st_col[s] + c, w = st_wave[s], st_tile_cur = st_tile[s];
      tma::mbar_wait(bar0 + 8 * s, phase);
      float2* sbuf = smem + F::OFF_CS + s * F::STAGE;
      const XformDesc d = a.desc[xf];
      const float2* dense = sbuf;
      fft::cta_fft<N, false, true, false, true, 2, F::COL_THREADS>(
          t, sbuf + c * F::CSTRIDE, stw, [&](int i) { return dense[i * PC + c]; },
          [&](int r, float2 x) {
            __stcs(d.out_re + (size_t)r * N + col, x.x);  // fft.cpp:93-99 split
            if (d.out_im) __stcs(d.out_im + (size_t)r * N + col, x.y);
          },
          [&] {
            named_sync<2, F::COL_THREADS>();  // the stage's shared reads are done
            if (leader) claim(s);
          });
      ++done_in_wave;
      const int tile_id = st_tile_cur;
      if (tile_id + (int)gridDim.x >= total_tiles || tile_id + (int)gridDim.x >= __ldg(a.tile0 + w + 1)) {
        // this CTA's last tile of wave w: release its reads to the row tasks
        named_sync<2, F::COL_THREADS>();
        if (leader) {
          __threadfence();
          atomicAdd(tiles_done + w, done_in_wave);
        }
        done_in_wave = 0;
      }
      if (++s == S) s = 0, phase ^= 1;
    }
  }
}
