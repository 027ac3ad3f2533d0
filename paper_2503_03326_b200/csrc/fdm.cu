// fdm.cu — Cords-Staadt interactive-wave zone (K9 mask + K10 stencil), sm_100a.
//
// Reference path replaced: FdmZone (interactive.cpp:33-129), compute_mask /
// point_in_loops / mask_height (interactive.cpp:21-31, 131-195), and the
// Simulation glue sim.cpp:86-109 (mask from the hydro waterline and volume).
//
// Scalar zone state (spacing, wave speed, damping, translation carry) is host
// bookkeeping exactly as in the reference; the fields live on the device as
// fp32 (curr / prev / next rotate). The mask arithmetic uses explicitly
// rounded fp64 intrinsics (no FMA contraction), so given the same loops the
// masked cell set is bit-identical to the reference.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "hydro_internal.cuh"
#include "spectrum_math.cuh"

namespace ocn {

ZoneView zone_view(ocn_zone* z) {
  ZoneView v;
  v.n = z->n;
  v.delta = z->delta;
  v.ox = z->origin[0];
  v.oz = z->origin[1];
  v.curr = z->curr();
  return v;
}

namespace {

// ---------------------------------------------------------------- K10 stencil
// next[i][j] = d (a lap(curr @ (i+wx, j+wz)) + 2 curr(i+wx, j+wz) - prev(i+ox, j+oz))
// (interactive.cpp:104-108); reads outside [0, n) are zero; margins stay zero.
// Each thread computes 4 consecutive cells of one row; interior threads (every
// read in range, the common case) take one branch-free path, the rest the
// bounds-checked one. Same arithmetic order in both.
struct FdmJob {
  int n, m, wx, wz, ox, oz;
  float a, d;
  const float* curr;
  const float* prev;
  float* next;
};
struct FdmBatch {
  int count;
  FdmJob j[kMaxBatch];
};

// zone blockIdx.z of the batch (every zone of a Simulation step in one launch)
__global__ void __launch_bounds__(256) k_fdm_step(const __grid_constant__ FdmBatch B) {
  const FdmJob& J = B.j[blockIdx.z];
  const int n = J.n, m = J.m, wx = J.wx, wz = J.wz, ox = J.ox, oz = J.oz;
  const float a = J.a, d = J.d;
  const float* __restrict__ curr = J.curr;
  const float* __restrict__ prev = J.prev;
  const int j0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int i = blockIdx.y;
  if (j0 >= n || i >= n) return;
  const int k = i + wx;
  const bool row_in = i >= m && i < n - m;
  const bool fast = row_in && k >= 1 && k + 1 < n && j0 >= m && j0 + 3 < n - m &&
                    j0 + wz >= 1 && j0 + 3 + wz + 1 < n && i + ox >= 0 && i + ox < n &&
                    j0 + oz >= 0 && j0 + 3 + oz < n;
  float out[4];
  if (fast) {
    const float* c0 = curr + (size_t)k * n + wz;
    const float* cm = c0 - n;
    const float* cp = c0 + n;
    const float* pr = prev + (size_t)(i + ox) * n + oz;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = j0 + q;
      const float ckl = __ldg(c0 + l);
      const float lap = __ldg(cp + l) + __ldg(cm + l) + __ldg(c0 + l + 1) + __ldg(c0 + l - 1) -
                        4.0f * ckl;
      out[q] = d * (a * lap + 2.0f * ckl - __ldg(pr + l));
    }
  } else {
    auto rd = [&](const float* f, int r, int c) {
      return (r < 0 || c < 0 || r >= n || c >= n) ? 0.f : __ldg(f + (size_t)r * n + c);
    };
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      out[q] = 0.f;
      if (row_in && j >= m && j < n - m) {
        const int l = j + wz;
        const float ckl = rd(curr, k, l);
        const float lap = rd(curr, k + 1, l) + rd(curr, k - 1, l) + rd(curr, k, l + 1) +
                          rd(curr, k, l - 1) - 4.0f * ckl;
        out[q] = d * (a * lap + 2.0f * ckl - rd(prev, i + ox, j + oz));
      }
    }
  }
  float* dst = J.next + (size_t)i * n + j0;
  if ((n & 3) == 0) {  // rows start 16-byte aligned: one vector store
    *reinterpret_cast<float4*>(dst) = make_float4(out[0], out[1], out[2], out[3]);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (j0 + q < n) dst[q] = out[q];
  }
}

__global__ void k_apply_cells(int n, int m, int count, const int* ij, const double* h, float* curr) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x) {
    const int i = ij[2 * q], j = ij[2 * q + 1];
    if (i < m || j < m || i >= n - m || j >= n - m) continue;
    curr[(size_t)i * n + j] = (float)h[q];
  }
}

// apply_mask (interactive.cpp:113-118) of the cell set the last mask pass
// left on the device (box [i0, i1) x [j0, j1), flags, heights); zone blockIdx.y
struct ApplyJob {
  const int* box;
  const unsigned char* mask_f;
  const double* mask_h;
  size_t cap;
  int n, m;
  float* curr;
};
struct ApplyBatch {
  int count;
  ApplyJob j[kMaxBatch];
};
__global__ void k_apply_box(const __grid_constant__ ApplyBatch B) {
  const ApplyJob& J = B.j[blockIdx.y];
  const int* box = J.box;
  const int i0 = box[0], i1 = box[1], j0 = box[2], j1 = box[3];
  if (box[4] <= 0 || i1 <= i0 || j1 <= j0) return;
  const int bw = j1 - j0, n = J.n, m = J.m;
  size_t cells = (size_t)(i1 - i0) * bw;
  if (cells > J.cap) cells = J.cap;
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < cells;
       c += (size_t)gridDim.x * blockDim.x) {
    if (!J.mask_f[c]) continue;
    const int i = i0 + (int)(c / bw), j = j0 + (int)(c % bw);
    if (i < m || j < m || i >= n - m || j >= n - m) continue;
    J.curr[(size_t)i * n + j] = (float)J.mask_h[c];
  }
}

__global__ void k_zone_sample(ZoneView z, int64_t count, const double* xz, double* out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = zone_sample(z, xz[2 * q], xz[2 * q + 1]);
}

__global__ void k_f32_f64(size_t n, const float* in, double* out) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x)
    out[q] = in[q];
}
__global__ void k_f64_f32(size_t n, const double* in, float* out) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x)
    out[q] = (float)in[q];
}

// ---------------------------------------------------------------- K9 mask
struct MaskArgs {
  double cy, sy;      // cos(-yaw), sin(-yaw) (host libm, as the reference)
  double bx, bz;      // body position
  double ox, oz, delta;
  int n, margin;
  double speed;
  ocn_mask_frame frame;
  ocn_mask_params params;
  const double* vw;   // device submerged volume (mask_from_hydro) or null
  double mesh_volume;
};

// One zone's mask pass (k_mask_prepare block / k_mask_cells grid row)
struct MaskJob {
  MaskArgs A;
  const int* nloops_dev;  // loop count on the device (mask_from_hydro) or null
  int nloops_host;
  const int* off;
  const double* pts;
  double* out_xz;
  int* out_off;
  double* bbox;
  int* box;
  int* bin_off;
  int* bin_edges;
  int bin_cap;
  int box_w_cap;
  double* mask_h;
  unsigned char* mask_f;
  float* curr;
  int apply;
  int* count;
};
struct MaskBatch {
  int count;
  MaskJob j[kMaxBatch];
};

__device__ __forceinline__ void derotate(const MaskArgs& A, double px, double pz, double* lx,
                                         double* lz) {
  const double qx = __dsub_rn(px, A.bx), qz = __dsub_rn(pz, A.bz);
  *lx = __dadd_rn(__dmul_rn(A.cy, qx), __dmul_rn(A.sy, qz));
  *lz = __dadd_rn(__dmul_rn(-A.sy, qx), __dmul_rn(A.cy, qz));
}

// One block: keep loops with >= 4 points (interactive.cpp:160), de-rotate them,
// loop bounding box, candidate cell box (interactive.cpp:172-181).
// loops: n_loops from *nloops_dev (or nloops_host when nloops_dev == null)
constexpr int kMaskBins = 1024;

__device__ __forceinline__ int mask_bin(double x, double lo, double w) {
  int b = (int)floor(__ddiv_rn(__dsub_rn(x, lo), w));
  return b < 0 ? 0 : (b >= kMaskBins ? kMaskBins - 1 : b);
}

// Edges binned by their x-range [min, max] (an edge can only change the +z
// ray parity of p when min(ax, bx) <= p.x < max(ax, bx)), so a cell tests the
// few edges of its bin; the per-edge test is untouched, so the parity (and the
// cell set) is exactly the reference's.
// zone blockIdx.x of the batch: one block per zone
__global__ void __launch_bounds__(1024) k_mask_prepare(const __grid_constant__ MaskBatch B) {
  const MaskJob& J = B.j[blockIdx.x];
  const MaskArgs& A = J.A;
  const int* off = J.off;
  const double* pts = J.pts;
  double* out_xz = J.out_xz;
  int* out_off = J.out_off;
  double* bbox = J.bbox;
  int* box = J.box;
  int* bin_off = J.bin_off;
  int* bin_edges = J.bin_edges;
  const int bin_cap = J.bin_cap;
  __shared__ int s_cnt[kMaskBins + 1];
  __shared__ int s_kept;
  __shared__ double s_lo[2][32], s_hi[2][32];
  __shared__ int s_wsum[32];
  const int nl = J.nloops_dev ? J.nloops_dev[0] : J.nloops_host;
  if (threadIdx.x == 0) {
    *J.count = 0;  // k_mask_cells accumulates into it
    int kept = 0, np = 0;
    out_off[0] = 0;
    for (int l = 0; l < nl; ++l) {
      const int c = off[l + 1] - off[l];
      if (c < 4) continue;
      np += c;
      out_off[++kept] = np;
    }
    s_kept = kept;
  }
  __syncthreads();
  const int kept = s_kept;
  double lox = 1e300, loz = 1e300, hix = -1e300, hiz = -1e300;
  // map kept loop k -> source loop
  int k = 0;
  for (int l = 0; l < nl; ++l) {
    const int c = off[l + 1] - off[l];
    if (c < 4) continue;
    const int dst = out_off[k];
    for (int q = threadIdx.x; q < c; q += blockDim.x) {
      double lx, lz;
      derotate(A, pts[3 * (off[l] + q)], pts[3 * (off[l] + q) + 2], &lx, &lz);
      out_xz[2 * (dst + q)] = lx;
      out_xz[2 * (dst + q) + 1] = lz;
      lox = lx < lox ? lx : lox;
      loz = lz < loz ? lz : loz;
      hix = hix < lx ? lx : hix;
      hiz = hiz < lz ? lz : hiz;
    }
    ++k;
  }
  // bbox: warp min / max, then across the warps (min / max are order-free)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lox = fmin(lox, __shfl_xor_sync(0xffffffffu, lox, o));
    loz = fmin(loz, __shfl_xor_sync(0xffffffffu, loz, o));
    hix = fmax(hix, __shfl_xor_sync(0xffffffffu, hix, o));
    hiz = fmax(hiz, __shfl_xor_sync(0xffffffffu, hiz, o));
  }
  if (lane == 0) s_lo[0][wid] = lox, s_lo[1][wid] = loz, s_hi[0][wid] = hix, s_hi[1][wid] = hiz;
  __syncthreads();
  if (wid == 0) {
    lox = lane < nw ? s_lo[0][lane] : 1e300;
    loz = lane < nw ? s_lo[1][lane] : 1e300;
    hix = lane < nw ? s_hi[0][lane] : -1e300;
    hiz = lane < nw ? s_hi[1][lane] : -1e300;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lox = fmin(lox, __shfl_xor_sync(0xffffffffu, lox, o));
      loz = fmin(loz, __shfl_xor_sync(0xffffffffu, loz, o));
      hix = fmax(hix, __shfl_xor_sync(0xffffffffu, hix, o));
      hiz = fmax(hiz, __shfl_xor_sync(0xffffffffu, hiz, o));
    }
    if (lane == 0) s_lo[0][0] = lox, s_lo[1][0] = loz, s_hi[0][0] = hix, s_hi[1][0] = hiz;
  }
  __syncthreads();
  const double lo_x = s_lo[0][0], hi_x = s_hi[0][0];
  double w = __ddiv_rn(__dsub_rn(hi_x, lo_x), (double)kMaskBins);
  if (!(w > 0.0)) w = 1.0;
  const int np = out_off[kept];
  auto edge_ok = [&](int q) {  // q -> q+1 inside one kept loop
    if (q + 1 >= np) return false;
    for (int l = 1; l <= kept; ++l)
      if (q + 1 == out_off[l]) return false;
    return true;
  };
  for (int b = threadIdx.x; b <= kMaskBins; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < np; q += blockDim.x) {
    if (!edge_ok(q)) continue;
    const double ax = out_xz[2 * q], bx = out_xz[2 * q + 2];
    const int b0 = mask_bin(fmin(ax, bx), lo_x, w), b1 = mask_bin(fmax(ax, bx), lo_x, w);
    for (int b = b0; b <= b1; ++b) atomicAdd(&s_cnt[b], 1);
  }
  __syncthreads();
  {  // exclusive scan of the bin counts (blockDim == kMaskBins == 1024)
    static_assert(kMaskBins == 1024, "one thread per bin");
    const int c = s_cnt[threadIdx.x];
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int wv = s_wsum[lane];
      int wi = wv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_wsum[lane] = wi - wv;
      if (lane == 31) s_cnt[kMaskBins] = wi, bin_off[kMaskBins] = wi;
    }
    __syncthreads();
    const int ex = s_wsum[wid] + incl - c;
    s_cnt[threadIdx.x] = ex;
    bin_off[threadIdx.x] = ex;
  }
  __syncthreads();
  const bool fits = s_cnt[kMaskBins] <= bin_cap;
  if (fits)
    for (int q = threadIdx.x; q < np; q += blockDim.x) {
      if (!edge_ok(q)) continue;
      const double ax = out_xz[2 * q], bx = out_xz[2 * q + 2];
      const int b0 = mask_bin(fmin(ax, bx), lo_x, w), b1 = mask_bin(fmax(ax, bx), lo_x, w);
      for (int b = b0; b <= b1; ++b) bin_edges[atomicAdd(&s_cnt[b], 1)] = q;
    }
  if (threadIdx.x != 0) return;
  bbox[0] = s_lo[0][0], bbox[1] = s_lo[1][0], bbox[2] = s_hi[0][0], bbox[3] = s_hi[1][0];
  bbox[4] = w;
  box[5] = fits ? 1 : 0;
  if (kept == 0) {
    box[0] = box[1] = box[2] = box[3] = 0;
    box[4] = 0;
    return;
  }
  const double ax = fmax(fabs(bbox[0]), fabs(bbox[2])), az = fmax(fabs(bbox[1]), fabs(bbox[3]));
  const double rad = sm::hypot_ref(ax, az);
  auto cell_of = [&](double w, double o) { return (int)floor(__ddiv_rn(__dsub_rn(w, o), A.delta)); };
  box[0] = max(A.margin, cell_of(__dsub_rn(A.bx, rad), A.ox));
  box[1] = min(A.n - A.margin, cell_of(__dadd_rn(A.bx, rad), A.ox) + 2);
  box[2] = max(A.margin, cell_of(__dsub_rn(A.bz, rad), A.oz));
  box[3] = min(A.n - A.margin, cell_of(__dadd_rn(A.bz, rad), A.oz) + 2);
  box[4] = kept;
}

// loop points cached in shared memory (16 KB: a mask CTA fits beside a
// column-pass CTA of a concurrent spectral step; longer waterlines read global)
constexpr int kMaskEdgesSmem = 1024;

// Per candidate cell: bbox cull, +z ray-crossing parity, V-shaped height;
// optionally writes the height into curr (apply_mask, interactive.cpp:113-118).
// zone blockIdx.y of the batch
__global__ void __launch_bounds__(256) k_mask_cells(const __grid_constant__ MaskBatch B) {
  const MaskJob& J = B.j[blockIdx.y];
  const MaskArgs& A = J.A;
  const int* box = J.box;
  const double* bbox = J.bbox;
  const int* loop_off = J.out_off;
  const double* loops_xz = J.out_xz;
  const int box_w_cap = J.box_w_cap;
  double* mask_h = J.mask_h;
  unsigned char* mask_f = J.mask_f;
  float* curr = J.curr;
  const int apply = J.apply;
  int* count = J.count;
  const int* bin_off = J.bin_off;
  const int* bin_edges = J.bin_edges;
  extern __shared__ double sm_pts[];
  const int i0 = box[0], i1 = box[1], j0 = box[2], j1 = box[3], kept = box[4];
  if (kept == 0 || i1 <= i0 || j1 <= j0) return;
  const int np = loop_off[kept];
  const bool cached = np <= kMaskEdgesSmem;
  for (int q = threadIdx.x; q < 2 * np && cached; q += blockDim.x) sm_pts[q] = loops_xz[q];
  __syncthreads();
  const double* P = cached ? sm_pts : loops_xz;
  const double lox = bbox[0], loz = bbox[1], hix = bbox[2], hiz = bbox[3], bw_x = bbox[4];
  const bool binned = box[5] != 0;
  double vr = A.frame.volume_ratio;
  if (A.vw) vr = A.mesh_volume > 0.0 ? __ddiv_rn(A.vw[0], A.mesh_volume) : 0.0;
  const int bw = j1 - j0;
  const long long cells = (long long)(i1 - i0) * bw;
  int local = 0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < cells;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = i0 + (int)(c / bw), j = j0 + (int)(c % bw);
    const double wx = __dadd_rn(A.ox, __dmul_rn((double)i, A.delta));
    const double wz = __dadd_rn(A.oz, __dmul_rn((double)j, A.delta));
    double lx, lz;
    derotate(A, wx, wz, &lx, &lz);
    unsigned char inside = 0;
    double h = 0.0;
    if (!(lx < lox || lx > hix || lz < loz || lz > hiz)) {
      int crossings = 0;
      auto test = [&](int e) {
        const double ax = P[2 * e], az = P[2 * e + 1], bx = P[2 * e + 2], bz = P[2 * e + 3];
        if ((ax > lx) == (bx > lx)) return;
        const double zi =
            __dadd_rn(az, __dmul_rn(__ddiv_rn(__dsub_rn(lx, ax), __dsub_rn(bx, ax)),
                                    __dsub_rn(bz, az)));
        if (zi > lz) ++crossings;
      };
      if (binned) {
        const int b = mask_bin(lx, lox, bw_x);
        for (int q = bin_off[b]; q < bin_off[b + 1]; ++q) test(bin_edges[q]);
      } else {
        for (int l = 0; l < kept; ++l)
          for (int e = loop_off[l]; e + 1 < loop_off[l + 1]; ++e) test(e);
      }
      if (crossings & 1) {
        inside = 1;
        // mask_height, interactive.cpp:21-31
        const ocn_mask_frame& F = A.frame;
        const double f = __ddiv_rn(fabs(__dsub_rn(lx, F.center_x)), F.half_beam);
        const double h_f = __dmul_rn(__dmul_rn(__dmul_rn(A.speed, F.mesh_height), A.params.intensity), vr);
        const double b_z = __dsub_rn(F.z_max, F.z_min);
        const double a = __ddiv_rn(__dsub_rn(h_f, A.params.back_height), b_z);
        const double b = __dsub_rn(A.params.back_height, __dmul_rn(a, F.z_min));
        h = __dmul_rn(A.params.amplitude, __dadd_rn(__dadd_rn(f, __dmul_rn(a, lz)), b));
        ++local;
        if (apply) curr[(size_t)i * A.n + j] = (float)h;
      }
    }
    if ((long long)c < (long long)box_w_cap) {
      mask_f[c] = inside;
      mask_h[c] = h;
    }
  }
  if (local) atomicAdd(count, local);
}

int blocks_for(ocn_ctx* ctx, size_t n, int threads = 256) {
  size_t b = (n + threads - 1) / threads;
  size_t cap = (size_t)ctx->sm_count * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

void check_mask_frame(const ocn_mask_frame* f) {
  if (!(f->half_beam > 0.0) || !(f->z_max > f->z_min))
    fail(OCN_ERR_DOMAIN, "mask_height: degenerate body frame");
}

// One zone's mask job (device buffers sized on the host first)
MaskJob mask_job(ocn_zone* z, const MaskArgs& A, const int* nloops_dev, int nloops_host,
                 const int* d_off, const double* d_pts, int max_points, int apply) {
  z->loops_xz.ensure(2 * (size_t)std::max(max_points, 1));
  z->loops_off.ensure((size_t)max_points / 4 + 2);
  const size_t box_cap = (size_t)(z->n - 2 * z->margin) * (z->n - 2 * z->margin);
  z->mask_h.ensure(box_cap);
  z->mask_f.ensure(box_cap);
  const int bin_cap = 8 * std::max(max_points, 1) + 16 * kMaskBins;
  z->bin_off.ensure(kMaskBins + 1);
  z->bin_edges.ensure(bin_cap);
  MaskJob J{};
  J.A = A;
  J.nloops_dev = nloops_dev;
  J.nloops_host = nloops_host;
  J.off = d_off;
  J.pts = d_pts;
  J.out_xz = z->loops_xz.p;
  J.out_off = z->loops_off.p;
  J.bbox = z->loop_bbox.p;
  J.box = z->mask_box.p;
  J.bin_off = z->bin_off.p;
  J.bin_edges = z->bin_edges.p;
  J.bin_cap = bin_cap;
  J.box_w_cap = (int)box_cap;
  J.mask_h = z->mask_h.p;
  J.mask_f = z->mask_f.p;
  J.curr = z->curr();
  J.apply = apply;
  J.count = z->mask_count.p;
  return J;
}

// the mask passes of B.count zones: two launches whatever the count
void mask_launch_batch(ocn_ctx* ctx, const MaskBatch& B) {
  NvtxRange nv("zones.mask");
  cudaStream_t st = ctx->stream;
  ProfWindow pw(ctx, OCN_PROF_MASK);
  k_mask_prepare<<<B.count, 1024, 0, st>>>(B);
  OCN_LAUNCHED(ctx);
  const size_t smem = kMaskEdgesSmem * 2 * sizeof(double);
  smem_opt_in(k_mask_cells, smem);
  const int per = std::max(1, ctx->sm_count * 4 / B.count);
  k_mask_cells<<<dim3(per, B.count), 256, smem, st>>>(B);
  OCN_LAUNCHED(ctx);
}

// shared by the explicit-loops and from-hydro entry points
void mask_launch(ocn_zone* z, MaskArgs A, const int* nloops_dev, int nloops_host,
                 const int* d_off, const double* d_pts, int max_points, int apply) {
  MaskBatch B{};
  B.count = 1;
  B.j[0] = mask_job(z, A, nloops_dev, nloops_host, d_off, d_pts, max_points, apply);
  mask_launch_batch(z->ctx, B);
}

MaskArgs mask_args(ocn_zone* z, double yaw, double bx, double bz, double speed,
                   const ocn_mask_frame* frame, const ocn_mask_params* params) {
  MaskArgs A{};
  A.cy = cos(-yaw);
  A.sy = sin(-yaw);
  A.bx = bx, A.bz = bz;
  A.ox = z->origin[0], A.oz = z->origin[1], A.delta = z->delta;
  A.n = z->n, A.margin = z->margin;
  A.speed = speed;
  A.frame = *frame;
  A.params = *params;
  return A;
}

}  // namespace

// FdmZone::step (interactive.cpp:67-111) of n zones: the scalar bookkeeping per
// zone on the host, the stencils as ONE launch (zone = blockIdx.z)
void zones_step_batch(int nz, ocn_zone* const* zones, double dt, const double* bx, const double* bz) {
  NvtxRange nv("zones.fdm");
  if (nz <= 0) return;
  OCN_REQUIRE(nz <= kMaxBatch, "%d zones in one step batch (max %d)", nz, kMaxBatch);
  ocn_ctx* ctx = zones[0]->ctx;
  FdmBatch B{};
  B.count = nz;
  int max_n = 0;
  for (int q = 0; q < nz; ++q) {
    ocn_zone* z = zones[q];
    OCN_REQUIRE(z && z->ctx == ctx, "zones must share one context");
    const double mx = bx[q] - z->pos_curr[0], mz = bz[q] - z->pos_curr[1];
    const double rx = mx / z->delta + z->carry[0];
    const double rz = mz / z->delta + z->carry[1];
    int wx = (int)std::floor(rx), wz = (int)std::floor(rz);
    z->carry[0] = rx - wx;
    z->carry[1] = rz - wz;
    const int max_shift = z->margin - 1;
    const size_t nn = (size_t)z->n * z->n;
    if (std::abs(wx) > max_shift || std::abs(wz) > max_shift) {
      wx = std::clamp(wx, -max_shift, max_shift);
      wz = std::clamp(wz, -max_shift, max_shift);
      OCN_CUDA(cudaMemsetAsync(z->curr(), 0, nn * sizeof(float), ctx->stream));
      OCN_CUDA(cudaMemsetAsync(z->prev(), 0, nn * sizeof(float), ctx->stream));
      ++z->dropped_wake;
    }
    const int ox = wx + z->last_shift[0], oz = wz + z->last_shift[1];
    const double a = z->c * z->c * dt * dt / (z->delta * z->delta);
    const int inext = 3 - z->icurr - z->iprev;
    B.j[q] = FdmJob{z->n, z->margin, wx, wz, ox, oz, (float)a, (float)z->damping,
                    z->curr(), z->prev(), z->buf[inext].p};
    max_n = std::max(max_n, z->n);
    z->iprev = z->icurr;
    z->icurr = inext;
    z->origin[0] += wx * z->delta;
    z->origin[1] += wz * z->delta;
    z->last_shift[0] = wx;
    z->last_shift[1] = wz;
    z->pos_curr[0] = bx[q];
    z->pos_curr[1] = bz[q];
  }
  const dim3 grid(((max_n + 3) / 4 + 255) / 256, max_n, nz);
  ProfWindow pw(ctx, OCN_PROF_FDM);
  k_fdm_step<<<grid, 256, 0, ctx->stream>>>(B);
  OCN_LAUNCHED(ctx);
}

// apply_mask (interactive.cpp:113-118) of each zone's last deferred mask, one launch
void zones_apply_last_mask_batch(int nz, ocn_zone* const* zones) {
  if (nz <= 0) return;
  OCN_REQUIRE(nz <= kMaxBatch, "%d zones in one mask batch (max %d)", nz, kMaxBatch);
  ocn_ctx* ctx = zones[0]->ctx;
  ApplyBatch B{};
  B.count = nz;
  for (int q = 0; q < nz; ++q) {
    ocn_zone* z = zones[q];
    OCN_REQUIRE(z && z->ctx == ctx, "zones must share one context");
    B.j[q] = ApplyJob{z->mask_box.p, z->mask_f.p, z->mask_h.p, z->mask_f.n, z->n, z->margin,
                      z->curr()};
  }
  k_apply_box<<<dim3(std::max(1, ctx->sm_count * 2 / nz), nz), 256, 0, ctx->stream>>>(B);
  OCN_LAUNCHED(ctx);
}

// Simulation's per-body masks (sim.cpp:86-99) from each mesh's last hydro
// evaluation, computed (not applied) for n zones in two launches
void zones_mask_from_hydro_batch(int nz, ocn_zone* const* zones, ocn_mesh* const* meshes,
                                 const double* yaw, const double* bx, const double* bz,
                                 const double* speed, const ocn_mask_frame* frames,
                                 const ocn_mask_params* params) {
  if (nz <= 0) return;
  OCN_REQUIRE(nz <= kMaxBatch, "%d zones in one mask batch (max %d)", nz, kMaxBatch);
  MaskBatch B{};
  B.count = nz;
  for (int q = 0; q < nz; ++q) {
    ocn_zone* z = zones[q];
    ocn_mesh* mesh = meshes[q];
    OCN_REQUIRE(z && mesh && frames && params, "bad arguments");
    OCN_REQUIRE(mesh->evaluated, "mesh has no hydro evaluation");
    OCN_REQUIRE(mesh->ctx == z->ctx && z->ctx == zones[0]->ctx, "meshes and zones must share one context");
    check_mask_frame(&frames[q]);
    MaskArgs A = mask_args(z, yaw[q], bx[q], bz[q], speed[q], &frames[q], &params[q]);
    A.vw = &mesh->report.p->r.submerged_volume;
    A.mesh_volume = mesh->volume;
    B.j[q] = mask_job(z, A, mesh->loop_counts.p, 0, mesh->loop_off.p, mesh->loop_points.p,
                      2 * mesh->nt + 2, 0);
  }
  mask_launch_batch(zones[0]->ctx, B);
}

}  // namespace ocn

using namespace ocn;

extern "C" {

int ocn_zone_create(ocn_ctx* ctx, const ocn_fdm_config* cfg, double body_size, double bx,
                    double bz, double dt, ocn_zone** out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && cfg && out, "null argument");
    if (cfg->grid_size < 8) fail(OCN_ERR_CONFIG, "FDM grid size too small");
    if (cfg->margin <= 1 || 2 * cfg->margin >= cfg->grid_size)
      fail(OCN_ERR_CONFIG, "FDM margin must satisfy 1 < m < grid_size/2");
    DeviceScope ds(ctx);
    auto z = std::make_unique<ocn_zone>();
    z->ctx = ctx;
    z->cfg = *cfg;
    z->n = cfg->grid_size;
    z->margin = cfg->margin;
    // interactive.cpp:36-51
    if (z->cfg.delta_min <= 0.0) z->cfg.delta_min = std::max(2.0 * body_size, 1e-3) / z->n;
    if (z->cfg.delta_max <= 0.0) z->cfg.delta_max = 10.0 * z->cfg.delta_min;
    if (z->cfg.delta_max < z->cfg.delta_min) fail(OCN_ERR_CONFIG, "FDM delta_max must be >= delta_min");
    const size_t nn = (size_t)z->n * z->n;
    for (auto& b : z->buf) {
      b.alloc(nn);
      OCN_CUDA(cudaMemsetAsync(b.p, 0, nn * sizeof(float), ctx->stream));
    }
    z->pos_curr[0] = bx, z->pos_curr[1] = bz;
    z->damping = cfg->d0;
    z->delta = std::clamp(0.999 * dt, z->cfg.delta_min, z->cfg.delta_max);
    z->c = std::sqrt(0.49) * z->delta / dt;
    z->origin[0] = bx - 0.5 * z->n * z->delta;
    z->origin[1] = bz - 0.5 * z->n * z->delta;
    z->mask_box.alloc(6);
    z->loop_bbox.alloc(5);
    z->mask_count.alloc(1);
    OCN_CUDA(cudaMemsetAsync(z->mask_box.p, 0, 6 * sizeof(int), ctx->stream));
    OCN_CUDA(cudaMemsetAsync(z->mask_count.p, 0, sizeof(int), ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx_retain(ctx);
    *out = z.release();
  });
}

int ocn_zone_destroy(ocn_zone* z) {
  if (!z) return OCN_OK;
  ocn_ctx* ctx = z->ctx;
  {
    DeviceScope ds(ctx);
    cudaStreamSynchronize(ctx->stream);
    delete z;
  }
  ctx_release(ctx);
  return OCN_OK;
}

int ocn_zone_get_state(const ocn_zone* z, ocn_zone_state* s) {
  if (!z || !s) return OCN_ERR_ARG;
  std::memset(s, 0, sizeof(*s));
  s->grid_size = z->n;
  s->margin = z->margin;
  s->spacing = z->delta;
  s->wave_speed = z->c;
  s->damping = z->damping;
  s->origin[0] = z->origin[0], s->origin[1] = z->origin[1];
  s->pos_curr[0] = z->pos_curr[0], s->pos_curr[1] = z->pos_curr[1];
  s->carry[0] = z->carry[0], s->carry[1] = z->carry[1];
  s->last_shift[0] = z->last_shift[0], s->last_shift[1] = z->last_shift[1];
  s->dropped_wake = z->dropped_wake;
  s->delta_min = z->cfg.delta_min;
  s->delta_max = z->cfg.delta_max;
  return OCN_OK;
}

// interactive.cpp:54-65
int ocn_zone_update_stability(ocn_zone* z, double speed, double dt) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z, "null zone");
    if (!(dt > 0.0)) fail(OCN_ERR_DOMAIN, "update_stability: dt must be > 0");
    double target = speed < 1.0 ? 0.999 * dt : speed * 0.999 * dt;
    target = std::clamp(target, z->cfg.delta_min, z->cfg.delta_max);
    const double lo = z->delta * (1.0 - z->cfg.delta_rate_limit);
    const double hi = z->delta * (1.0 + z->cfg.delta_rate_limit);
    z->delta = std::clamp(target, lo, hi);
    z->delta = std::clamp(z->delta, z->cfg.delta_min, z->cfg.delta_max);
    z->c = std::sqrt(0.49) * z->delta / dt;
    z->damping = sm::damping_factor(speed, z->cfg.d0, z->cfg.d_max, z->cfg.v_max);
  });
}

// interactive.cpp:67-111
int ocn_zone_step(ocn_zone* z, double dt, double bx, double bz) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z, "null zone");
    DeviceScope ds(z->ctx);
    zones_step_batch(1, &z, dt, &bx, &bz);
  });
}

int ocn_zone_apply_cells(ocn_zone* z, int count, const int32_t* ij, const double* h) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z && count >= 0 && (count == 0 || (ij && h)), "bad arguments");
    if (count == 0) return;
    ocn_ctx* ctx = z->ctx;
    DeviceScope ds(ctx);
    DevBuf<int> dij(2 * (size_t)count);
    DevBuf<double> dh(count);
    OCN_CUDA(cudaMemcpyAsync(dij.p, ij, 2 * (size_t)count * sizeof(int), cudaMemcpyHostToDevice,
                             ctx->stream));
    OCN_CUDA(cudaMemcpyAsync(dh.p, h, (size_t)count * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    k_apply_cells<<<blocks_for(ctx, count), 256, 0, ctx->stream>>>(z->n, z->margin, count, dij.p,
                                                                   dh.p, z->curr());
    OCN_LAUNCHED(ctx);
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ocn_zone_compute_mask(ocn_zone* z, int n_loops, const int32_t* off, const double* pts,
                          double yaw, double bx, double bz, double speed,
                          const ocn_mask_frame* frame, const ocn_mask_params* params, int apply,
                          int* n_cells) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z && frame && params && (n_loops == 0 || (off && pts)), "bad arguments");
    ocn_ctx* ctx = z->ctx;
    DeviceScope ds(ctx);
    int total = n_loops > 0 ? off[n_loops] : 0;
    bool any = false;
    for (int l = 0; l < n_loops; ++l) any |= (off[l + 1] - off[l]) >= 4;
    if (any) check_mask_frame(frame);
    DevBuf<int> doff((size_t)n_loops + 1);
    DevBuf<double> dpts(3 * (size_t)std::max(total, 1));
    if (n_loops > 0) {
      OCN_CUDA(cudaMemcpyAsync(doff.p, off, ((size_t)n_loops + 1) * sizeof(int),
                               cudaMemcpyHostToDevice, ctx->stream));
      OCN_CUDA(cudaMemcpyAsync(dpts.p, pts, 3 * (size_t)total * sizeof(double),
                               cudaMemcpyHostToDevice, ctx->stream));
    }
    MaskArgs A = mask_args(z, yaw, bx, bz, speed, frame, params);
    mask_launch(z, A, nullptr, n_loops, doff.p, dpts.p, total, apply);
    int cnt = 0;
    OCN_CUDA(cudaMemcpyAsync(&cnt, z->mask_count.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    if (n_cells) *n_cells = cnt;
  });
}

int ocn_zone_mask_from_hydro(ocn_zone* z, ocn_mesh* mesh, double yaw, double bx, double bz,
                             double speed, const ocn_mask_frame* frame,
                             const ocn_mask_params* params) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z && mesh && frame && params, "bad arguments");
    OCN_REQUIRE(mesh->evaluated, "mesh has no hydro evaluation");
    OCN_REQUIRE(mesh->ctx == z->ctx, "mesh and zone use different contexts");
    check_mask_frame(frame);
    DeviceScope ds(z->ctx);
    MaskArgs A = mask_args(z, yaw, bx, bz, speed, frame, params);
    A.vw = &mesh->report.p->r.submerged_volume;
    A.mesh_volume = mesh->volume;
    mask_launch(z, A, mesh->loop_counts.p, 0, mesh->loop_off.p, mesh->loop_points.p,
                2 * mesh->nt + 2, 1);
  });
}

int ocn_zone_mask_from_hydro_deferred(ocn_zone* z, ocn_mesh* mesh, double yaw, double bx, double bz,
                                      double speed, const ocn_mask_frame* frame,
                                      const ocn_mask_params* params) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z && mesh && frame && params, "bad arguments");
    OCN_REQUIRE(mesh->evaluated, "mesh has no hydro evaluation");
    OCN_REQUIRE(mesh->ctx == z->ctx, "mesh and zone use different contexts");
    check_mask_frame(frame);
    DeviceScope ds(z->ctx);
    MaskArgs A = mask_args(z, yaw, bx, bz, speed, frame, params);
    A.vw = &mesh->report.p->r.submerged_volume;
    A.mesh_volume = mesh->volume;
    mask_launch(z, A, mesh->loop_counts.p, 0, mesh->loop_off.p, mesh->loop_points.p,
                2 * mesh->nt + 2, 0);
  });
}

int ocn_zone_apply_last_mask(ocn_zone* z) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z, "null zone");
    DeviceScope ds(z->ctx);
    zones_apply_last_mask_batch(1, &z);
  });
}

int ocn_zone_mask_download(ocn_zone* z, int capacity, int32_t* ij, double* h, int* n_cells) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z, "null zone");
    ocn_ctx* ctx = z->ctx;
    DeviceScope ds(ctx);
    OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    int box[5];
    OCN_CUDA(cudaMemcpy(box, z->mask_box.p, sizeof(box), cudaMemcpyDeviceToHost));
    int cnt = 0;
    if (box[4] > 0 && box[1] > box[0] && box[3] > box[2]) {
      const size_t cells = (size_t)(box[1] - box[0]) * (box[3] - box[2]);
      std::vector<unsigned char> f(cells);
      std::vector<double> hh(cells);
      OCN_CUDA(cudaMemcpy(f.data(), z->mask_f.p, cells, cudaMemcpyDeviceToHost));
      OCN_CUDA(cudaMemcpy(hh.data(), z->mask_h.p, cells * sizeof(double), cudaMemcpyDeviceToHost));
      const int bw = box[3] - box[2];
      for (size_t c = 0; c < cells; ++c) {
        if (!f[c]) continue;
        if (cnt < capacity) {
          if (ij) ij[2 * cnt] = box[0] + (int)(c / bw), ij[2 * cnt + 1] = box[2] + (int)(c % bw);
          if (h) h[cnt] = hh[c];
        }
        ++cnt;
      }
    }
    if (n_cells) *n_cells = cnt;
  });
}

int ocn_zone_sample(ocn_zone* z, int64_t count, const double* xz, double* out) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z && count >= 0 && (count == 0 || (xz && out)), "bad arguments");
    if (count == 0) return;
    ocn_ctx* ctx = z->ctx;
    DeviceScope ds(ctx);
    InStage si(ctx, xz, (size_t)count * 2 * sizeof(double));
    OutStage so(ctx, out, (size_t)count * sizeof(double));
    k_zone_sample<<<blocks_for(ctx, count), 256, 0, ctx->stream>>>(zone_view(z), count,
                                                                   (const double*)si.dev,
                                                                   (double*)so.dev);
    OCN_LAUNCHED(ctx);
    so.finish();
  });
}

int ocn_zone_download(ocn_zone* z, double* curr, double* prev) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z, "null zone");
    ocn_ctx* ctx = z->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)z->n * z->n;
    DevBuf<double> tmp(nn);
    for (int k = 0; k < 2; ++k) {
      double* dst = k == 0 ? curr : prev;
      if (!dst) continue;
      k_f32_f64<<<blocks_for(ctx, nn), 256, 0, ctx->stream>>>(nn, k == 0 ? z->curr() : z->prev(),
                                                              tmp.p);
      OCN_LAUNCHED(ctx);
      OCN_CUDA(cudaMemcpyAsync(dst, tmp.p, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

int ocn_zone_upload(ocn_zone* z, const double* curr, const double* prev) {
  return api_call(z ? z->ctx : nullptr, [&] {
    OCN_REQUIRE(z, "null zone");
    ocn_ctx* ctx = z->ctx;
    DeviceScope ds(ctx);
    const size_t nn = (size_t)z->n * z->n;
    DevBuf<double> tmp(nn);
    for (int k = 0; k < 2; ++k) {
      const double* src = k == 0 ? curr : prev;
      if (!src) continue;
      OCN_CUDA(cudaMemcpyAsync(tmp.p, src, nn * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      k_f64_f32<<<blocks_for(ctx, nn), 256, 0, ctx->stream>>>(nn, tmp.p,
                                                              k == 0 ? z->curr() : z->prev());
      OCN_LAUNCHED(ctx);
      OCN_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

}  // extern "C"
