// hydro.cu — fluid-to-solid forces on a triangle hull (K5-K8), sm_100a.
//
// Reference path replaced: classify_clip (hydro.cpp:63-215), submerged_volume
// (:217-223), center_of_immersion (:225-238), buoyancy (:240), drag (:242-251),
// aggregate (:253-306) with the Simulation samplers (sim.cpp:39-51, 74-83).
//
// Pipeline (one stream, no host round trip until the report is read):
//   k_vertices   world transform + Algorithm-1 height (+ other zones) -> depth
//   k_classify_scan  per triangle: 0 / 1 / 3 states, 0 / 1 waterline segment,
//                and the block-local exclusive scan of those counts
//   (last classify block) the block totals -> order-preserving offsets (parent
//                order, hydro.cpp:151-163)
//   k_emit       TriangleStates and crossing segments at their offsets
//   k_forces     per state: prism volume, immersion moment, drag (velocity_at
//                at the centroid), dry area / moment -> fixed-tree block sums;
//                the last block (ticket) reduces them in a fixed order, clamps,
//                buoyancy, application points, composed force / torque
//                (sim.cpp:114-122)
//   k_chain      waterline chaining with the reference's visiting order
//                (hydro.cpp:165-213): start at the lowest unused segment,
//                enter through its first edge, last-writer crossing points.
// All reductions are fixed trees over a fixed state->thread mapping, so the
// report is bit-identical run to run.
#include <algorithm>
#include <cstring>
#include <vector>

#include "hydro_internal.cuh"
#include "samplers.cuh"

namespace ocn {
namespace {

__device__ __forceinline__ double3 d3(double x, double y, double z) { return make_double3(x, y, z); }
__device__ __forceinline__ double3 operator+(double3 a, double3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ double3 operator-(double3 a, double3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double3 operator*(double3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ double3 cross3(double3 a, double3 b) {
  return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double dot3(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double norm3(double3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
__device__ __forceinline__ double3 ld3(const double* p) { return d3(p[0], p[1], p[2]); }
__device__ __forceinline__ void st3(double* p, double3 v) { p[0] = v.x, p[1] = v.y, p[2] = v.z; }

// Quat::rotate (core.hpp:164-169)
__device__ __forceinline__ double3 qrot(const PoseDev& P, double3 v) {
  const double3 u = d3(P.q[1], P.q[2], P.q[3]);
  const double3 t = cross3(u, v) * 2.0;
  return (v + t * P.q[0]) + cross3(u, t);
}

// ---------------------------------------------------------------- K5: vertices
// Four lanes per vertex: lane q sums the cascades c = q, q + 4, ... of each
// Algorithm-1 iteration (surface.cpp:141-151, 4 iterations) and the four
// partials are combined by a fixed xor tree, so the 48 taps of an iteration
// are in flight together and 4x more threads hide the gather latency.
template <int NB>
__global__ void __launch_bounds__(128) k_vertices(const __grid_constant__ HydroBatch<NB> B) {
  const HydroJob& J = B.job[blockIdx.y];
  const int nv = J.nv;
  const double* __restrict__ verts = J.verts;
  const PoseDev& P = J.P;
  const SurfView& surf = B.surf;
  const int have_surf = B.have_surf;
  const ZoneList& zones = J.zones;
  const double* override_depth = J.override_depth;
  double* wpos = J.wpos;
  double* depth = J.depth;
  {  // the evaluation's resets (read only by later kernels): flags, waterline hash table
    const int i0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    if (i0 < 4) J.flags[i0] = 0;
    for (int i = i0; i < J.hcap; i += stride) J.hkeys[i] = 0ull;
    for (int i = i0; i < 3 * J.hcap; i += stride) J.hvals[i] = 0;
  }
  const int lane = threadIdx.x & 31, q = lane & 3;
  const int per_warp = 8;  // vertices per warp pass
  const int warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int base = warp_g * per_warp; base < nv; base += warps * per_warp) {
    const int iv = base + (lane >> 2);
    const bool valid = iv < nv;
    const int i = valid ? iv : nv - 1;  // every lane takes part in the shuffles
    const double3 b = ld3(verts + 3 * i);
    const double3 w = d3(P.p[0], P.p[1], P.p[2]) + qrot(P, b - d3(P.com[0], P.com[1], P.com[2]));
    double d;
    if (override_depth) {
      d = override_depth[i];
    } else {
      double h = 0.0;
      if (have_surf) {
        double wx = 0.0, wz = 0.0;
#pragma unroll 1
        for (int it = 0; it < 4; ++it) {
          const double qx = w.x - wx, qz = w.z - wz;
          double sx = 0.0, sh = 0.0, sz = 0.0;
          for (int c = q; c < surf.C; c += 4) {
            const Bilin bl = bilin_setup(surf.n, surf.length[c], qx, qz);
            sx += bilin_tap(bl, surf.f(c, OCN_FIELD_DX));
            sh += bilin_tap(bl, surf.f(c, OCN_FIELD_H));
            sz += bilin_tap(bl, surf.f(c, OCN_FIELD_DZ));
          }
#pragma unroll
          for (int o = 1; o < 4; o <<= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sh += __shfl_xor_sync(0xffffffffu, sh, o);
            sz += __shfl_xor_sync(0xffffffffu, sz, o);
          }
          wx = sx, wz = sz, h = sh;
        }
      }
      for (int z = 0; z < zones.count; ++z) h += zone_sample(zones.z[z], w.x, w.z);
      d = w.y - h;
    }
    if (valid && q == 0) {
      st3(wpos + 3 * i, w);
      depth[i] = d;
    }
  }
}

// ---------------------------------------------------------------- K7: classify + scan
// counts.x = states emitted (0 degenerate, 1 whole, 3 split), counts.y = segment.
// One triangle per thread; each 1024-triangle block also scans its counts
// (exclusive, parent order, hydro.cpp:151-163) and leaves its total for
// the last classify block; k_emit adds the block's offset.
constexpr int kScanBlock = 512;  // <= 16 K registers per CTA: fits beside a column-pass CTA

__device__ __forceinline__ int2 add2(int2 a, int2 b) { return make_int2(a.x + b.x, a.y + b.y); }

// exclusive scan of one int2 per thread over a block of kScanBlock threads
// (warp shuffles, then the 32 warp totals by warp 0)
__device__ int2 block_exclusive_scan(int2 v, int2* warp_tot, int2* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int2 incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, incl.x, off);
    const int y = __shfl_up_sync(0xffffffffu, incl.y, off);
    if (lane >= off) incl.x += x, incl.y += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int2 w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : make_int2(0, 0);
    int2 wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, wi.x, off);
      const int y = __shfl_up_sync(0xffffffffu, wi.y, off);
      if (lane >= off) wi.x += x, wi.y += y;
    }
    warp_tot[lane] = make_int2(wi.x - w.x, wi.y - w.y);  // exclusive warp offsets
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const int2 base = warp_tot[warp];
  return make_int2(base.x + incl.x - v.x, base.y + incl.y - v.y);
}

template <int NB>
__global__ void __launch_bounds__(kScanBlock) k_classify_scan(const __grid_constant__ HydroBatch<NB> B) {
  const HydroJob& J = B.job[blockIdx.y];
  const int nt = J.nt;
  if ((int)blockIdx.x * kScanBlock >= nt) return;  // this job's blocks end earlier (uniform)
  const int3* __restrict__ tris = J.tris;
  const double* __restrict__ areas = J.areas;
  const double* __restrict__ depth = J.depth;
  int2* counts = J.counts;
  int2* offsets = J.offsets;
  int2* block_sums = J.block_sums;
  __shared__ int2 warp_tot[32];
  __shared__ int2 tot;
  const int t = blockIdx.x * kScanBlock + threadIdx.x;
  int2 c = make_int2(0, 0);
  if (t < nt && areas[t] > 0.0) {
    const int3 v = tris[t];
    const int above = (depth[v.x] >= 0.0) + (depth[v.y] >= 0.0) + (depth[v.z] >= 0.0);
    if (above == 0 || above == 3) {
      c.x = 1;
    } else {
      c.x = 3;
      c.y = 1;  // keys (a,b) != (a,c) since a, b, c are distinct in a validated mesh
    }
  }
  const int2 ex = block_exclusive_scan(c, warp_tot, &tot);
  if (t < nt) {
    counts[t] = c;
    offsets[t] = ex;
  }
  __syncthreads();
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
  // the last of this job's blocks scans the block totals (was k_scan_blocks);
  // the ticket is k_forces' too, each resetting it when done
  const int nb = (nt + kScanBlock - 1) / kScanBlock;
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(J.ticket, 1) == nb - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  int2 carry = make_int2(0, 0);
  for (int base = 0; base < nb; base += kScanBlock) {
    const int i = base + threadIdx.x;
    const int2 v = i < nb ? __ldcg(block_sums + i) : make_int2(0, 0);
    const int2 bex = block_exclusive_scan(v, warp_tot, &tot);
    if (i < nb) block_sums[i] = add2(carry, bex);
    __syncthreads();
    carry = add2(carry, tot);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *J.total = carry;
    *J.ticket = 0;
  }
}


// ---------------------------------------------------------------- K7: emit
__device__ __forceinline__ void emit_state(StateDev* s, int parent, int status, double3 a, double3 b,
                                           double3 c, double da, double db, double dc, double3 n) {
  StateDev r;
  r.parent = parent;
  r.status = status;
  r.area = 0.5 * norm3(cross3(b - a, c - a));
  // (a + b + c) / 3 as the reference divides (hydro.cpp:47)
  r.centroid = d3(((a.x + b.x) + c.x) / 3.0, ((a.y + b.y) + c.y) / 3.0, ((a.z + b.z) + c.z) / 3.0);
  r.depth = (da + db + dc) / 3.0;
  r.normal = n;
  *s = r;
}

template <int NB>
__global__ void __launch_bounds__(128) k_emit(const __grid_constant__ HydroBatch<NB> B) {
  const HydroJob& J = B.job[blockIdx.y];
  const int nt = J.nt;
  const int3* __restrict__ tris = J.tris;
  const double* __restrict__ normals = J.normals;
  const double* __restrict__ wpos = J.wpos;
  const double* __restrict__ depth = J.depth;
  const PoseDev& P = J.P;
  const int2* __restrict__ counts = J.counts;
  const int2* __restrict__ offsets = J.offsets;
  const int2* __restrict__ block_sums = J.block_sums;
  StateDev* states = J.states;
  SegDev* segs = J.segs;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const int2 c = counts[t];
    if (c.x == 0) continue;
    const int2 off = add2(offsets[t], block_sums[t / kScanBlock]);
    const int3 v = tris[t];
    const double3 n = qrot(P, ld3(normals + 3 * t));
    const double d0 = depth[v.x], d1 = depth[v.y], d2 = depth[v.z];
    if (c.x == 1) {
      const int status = d0 >= 0.0 ? 1 : 0;  // all above -> Dry (1), all below -> Submerged (0)
      emit_state(states + off.x, t, status, ld3(wpos + 3 * v.x), ld3(wpos + 3 * v.y),
                 ld3(wpos + 3 * v.z), d0, d1, d2, n);
      continue;
    }
    const bool ab0 = d0 >= 0.0, ab1 = d1 >= 0.0, ab2 = d2 >= 0.0;
    const int above = ab0 + ab1 + ab2;
    int a, b, cc;
    bool odd_above;
    if (above == 1) {
      odd_above = true;
      if (ab0) a = v.x, b = v.y, cc = v.z;
      else if (ab1) a = v.y, b = v.z, cc = v.x;
      else a = v.z, b = v.x, cc = v.y;
    } else {
      odd_above = false;
      if (!ab0) a = v.x, b = v.y, cc = v.z;
      else if (!ab1) a = v.y, b = v.z, cc = v.x;
      else a = v.z, b = v.x, cc = v.y;
    }
    const double da = depth[a], db = depth[b], dc = depth[cc];
    const double alpha_ab = da / (da - db);
    const double alpha_ac = da / (da - dc);
    const double3 wa = ld3(wpos + 3 * a), wb = ld3(wpos + 3 * b), wc = ld3(wpos + 3 * cc);
    const double3 pab = wa + (wb - wa) * alpha_ab;
    const double3 pac = wa + (wc - wa) * alpha_ac;
    const int odd_status = odd_above ? 1 : 0, rest = odd_above ? 0 : 1;
    emit_state(states + off.x, t, odd_status, wa, pab, pac, da, 0.0, 0.0, n);
    emit_state(states + off.x + 1, t, rest, pab, wb, wc, 0.0, db, dc, n);
    emit_state(states + off.x + 2, t, rest, pab, wc, pac, 0.0, dc, 0.0, n);
    SegDev s;
    s.ka = make_int2(min(a, b), max(a, b));
    s.kb = make_int2(min(a, cc), max(a, cc));
    s.pa = pab;
    s.pb = pac;
    segs[off.y] = s;
  }
}

// ---------------------------------------------------------------- K6 + K8: forces
// Per-state terms accumulated per thread over a fixed strided set of states,
// then a fixed shared-memory tree. Slots (all fp64):
//  0 v_w   1 cw   2..4 moment   5..7 F_w/rho   8..10 F_a   11 dry area
//  12..14 dry moment   15 submerged area   16 nonfinite count
constexpr int kTerms = 17;
constexpr int kForceThreads = 256;

__device__ __forceinline__ double3 drag_dev(const StateDev& s, double3 medium, double rho,
                                            double cd, const PoseDev& P) {
  const double3 pos = d3(P.p[0], P.p[1], P.p[2]);
  const double3 vpt = d3(P.v[0], P.v[1], P.v[2]) + cross3(d3(P.w[0], P.w[1], P.w[2]), s.centroid - pos);
  const double3 vrel = vpt - medium;
  const double speed = norm3(vrel);
  if (speed < 1e-12 || s.area <= 0.0) return d3(0, 0, 0);
  const double facing = dot3(s.normal, d3(vrel.x / speed, vrel.y / speed, vrel.z / speed));
  if (facing <= 0.0) return d3(0, 0, 0);
  const double a_perp = s.area * facing;
  return vrel * (-(0.5 * cd * rho * a_perp * speed));
}

__device__ void finalize_report(int nblocks, const double* block_out, PoseDev P, FluidDev F,
                                double mesh_volume, const int2* total, int degenerate,
                                ReportDev* rep);

// Per-state loads (hydro.cpp:215-306) reduced per block in a fixed tree; the
// last block to finish (ticket counter) reduces the block partials in a fixed
// order and writes the report, so no separate finalize launch is needed.
template <int NB>
__global__ void __launch_bounds__(kForceThreads) k_forces(const __grid_constant__ HydroBatch<NB> B) {
  const HydroJob& J = B.job[blockIdx.y];
  const StateDev* __restrict__ states = J.states;
  const int2* total = J.total;
  const PoseDev& P = J.P;
  const SliceView& vel = B.vel;
  const int have_vel = B.have_vel, clamp = J.clamp;
  const FluidDev& F = J.F;
  double* block_out = J.block_out;
  int* domain_err = J.flags;
  int* ticket = J.ticket;
  const double mesh_volume = J.volume;
  const int degenerate = J.degenerate;
  ReportDev* rep = J.report;
  const double* __restrict__ ext_vel = J.ext_vel;
  __shared__ double wsum[kForceThreads / 32][kTerms];
  const int ns = total->x;
  double acc[kTerms];
#pragma unroll
  for (int k = 0; k < kTerms; ++k) acc[k] = 0.0;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride) {
    const StateDev s = states[i];
    if (s.status == 0) {
      const double w = s.area * s.depth * s.normal.y;
      acc[0] += w;
      acc[1] += w;
      acc[2] += s.centroid.x * w;
      acc[3] += (s.centroid.y - 0.5 * s.depth) * w;
      acc[4] += s.centroid.z * w;
      double3 med = d3(0, 0, 0);
      if (ext_vel) {  // host sampler results, one triple per state
        med = d3(ext_vel[3 * i], ext_vel[3 * i + 1], ext_vel[3 * i + 2]);
      } else if (have_vel) {
        double v[3];
        if (!velocity_at_dev(vel, s.centroid.x, s.centroid.z, s.centroid.y, OCN_INTERP_EXPONENTIAL,
                             clamp, v))
          atomicOr(domain_err, 1);
        med = d3(v[0], v[1], v[2]);
      }
      const double3 f = drag_dev(s, med, 1.0, F.cd_water, P);  // rho_w applied at finalize
      acc[5] += f.x, acc[6] += f.y, acc[7] += f.z;
      acc[15] += s.area;
    } else {
      const double3 f = drag_dev(s, d3(F.wind[0], F.wind[1], F.wind[2]), F.air_density, F.cd_air, P);
      acc[8] += f.x, acc[9] += f.y, acc[10] += f.z;
      acc[11] += s.area;
      acc[12] += s.centroid.x * s.area;
      acc[13] += s.centroid.y * s.area;
      acc[14] += s.centroid.z * s.area;
    }
  }
  // fixed tree: xor shuffles within each warp, then the warps in order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kTerms - 1; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) wsum[warp][k] = v;
  }
  if (lane == 0) wsum[warp][kTerms - 1] = 0.0;
  __syncthreads();
  if (threadIdx.x < kTerms) {
    double v = 0.0;
    for (int w = 0; w < kForceThreads / 32; ++w) v += wsum[w][threadIdx.x];
    block_out[blockIdx.x * kTerms + threadIdx.x] = v;
  }
  __threadfence();  // this block's partials, before its ticket
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_report(gridDim.x, block_out, P, F, mesh_volume, total, degenerate, rep);
  if (threadIdx.x == 0) *ticket = 0;  // ready for the next evaluation
}

__device__ __forceinline__ double density_at_dev(const FluidDev& F, double y) {
  const int n = F.n_profile;
  const double* p = F.profile;
  if (n == 0) return F.water_density;
  if (y <= p[0]) return p[1];
  if (y >= p[2 * (n - 1)]) return p[2 * (n - 1) + 1];
  for (int i = 1; i < n; ++i)
    if (y <= p[2 * i]) {
      const double y0 = p[2 * (i - 1)], r0 = p[2 * (i - 1) + 1], y1 = p[2 * i], r1 = p[2 * i + 1];
      const double u = (y - y0) / (y1 - y0);
      return (1.0 - u) * r0 + u * r1;
    }
  return F.water_density;
}

__device__ __forceinline__ bool finite3(double3 v) {
  return isfinite(v.x) && isfinite(v.y) && isfinite(v.z);
}

// one block: fixed-order tree over the block partials, then the report
// Block partials -> totals (one warp per term: lane-strided sums in block
// order, then a fixed xor tree), then the report (hydro.cpp:215-306,
// sim.cpp:114-122). Called by the last k_forces block (kForceThreads threads).
__device__ void finalize_report(int nblocks, const double* block_out, PoseDev P, FluidDev F,
                                double mesh_volume, const int2* total, int degenerate,
                                ReportDev* rep) {
  __shared__ double tot[kTerms][1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
  for (int k = warp; k < kTerms; k += warps) {
    double a = 0.0;
    for (int b = lane; b < nblocks; b += 32) a += __ldcg(block_out + b * kTerms + k);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if (lane == 0) tot[k][0] = a;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto sh = tot;
  ocn_hydro_report r;
  memset(&r, 0, sizeof(r));
  double vw = sh[0][0];
  if (vw < 0.0) {
    vw = 0.0;
    r.volume_clamped = 1;
  } else if (vw > mesh_volume) {
    vw = mesh_volume;
    r.volume_clamped = 1;
  }
  r.submerged_volume = vw;
  const double cw = sh[1][0];
  const double3 pos = d3(P.p[0], P.p[1], P.p[2]);
  double3 coi = d3(0, 0, 0);
  r.has_center_of_immersion = cw > 1e-12;
  if (r.has_center_of_immersion) coi = d3(sh[2][0] / cw, sh[3][0] / cw, sh[4][0] / cw);
  double rho_w = F.water_density;
  if (F.n_profile > 0 && r.has_center_of_immersion) rho_w = density_at_dev(F, coi.y);
  const double3 fw = d3(sh[5][0] * rho_w, sh[6][0] * rho_w, sh[7][0] * rho_w);
  const double3 fa = d3(sh[8][0], sh[9][0], sh[10][0]);
  double3 fb = d3(0, 0, 0), wc = pos;
  if (r.has_center_of_immersion) {
    fb = d3(0.0 * -(vw * rho_w), -kGravity * -(vw * rho_w), 0.0 * -(vw * rho_w));  // hydro.cpp:240, 290
    wc = coi;
  }
  const double dry = sh[11][0];
  const double3 ac = dry > 1e-12 ? d3(sh[12][0] / dry, sh[13][0] / dry, sh[14][0] / dry) : pos;
  double3 Ft = d3(0, 0, 0), T = d3(0, 0, 0);
  if (r.has_center_of_immersion) {
    Ft = Ft + fb;
    T = T + cross3(wc - pos, fb);
    Ft = Ft + fw;
    T = T + cross3(wc - pos, fw);
  }
  Ft = Ft + fa;
  T = T + cross3(ac - pos, fa);
  st3(r.center_of_immersion, coi);
  st3(r.buoyancy_force, fb);
  st3(r.water_drag, fw);
  st3(r.air_drag, fa);
  st3(r.water_center, wc);
  st3(r.air_center, ac);
  r.submerged_area = sh[15][0];
  r.dry_area = dry;
  st3(r.force, Ft);
  st3(r.torque, T);
  r.state_count = total->x;
  r.degenerate_skipped = degenerate;
  r.nonfinite = !(isfinite(vw) && finite3(coi) && finite3(fw) && finite3(fa) && finite3(Ft) &&
                  finite3(T) && finite3(ac));
  rep->r = r;
}

// ---------------------------------------------------------------- waterline chaining
__device__ __forceinline__ unsigned long long key64(int2 k) {
  return ((unsigned long long)(unsigned)k.x << 32) | (unsigned)k.y;
}
__device__ __forceinline__ unsigned hash64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return (unsigned)k;
}

// Inserts every (segment, side) under its edge key; a key on a closed mesh
// has exactly two entries (the two triangles sharing the crossed edge).
template <int NB>
__global__ void k_chain_hash(const __grid_constant__ HydroBatch<NB> B) {
  const HydroJob& J = B.job[blockIdx.y];
  const SegDev* segs = J.segs;
  const int2* total = J.total;
  const int hcap = J.hcap;
  unsigned long long* hkeys = J.hkeys;
  int* hvals = J.hvals;
  int* err = J.flags + 1;
  const int nseg = total->y;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * nseg; e += gridDim.x * blockDim.x) {
    const int s = e >> 1, side = e & 1;
    const int2 k = side ? segs[s].kb : segs[s].ka;
    const unsigned long long key = key64(k) + 1ull;
    unsigned h = hash64(key) & (hcap - 1);
    for (int probe = 0; probe < hcap; ++probe) {
      const unsigned long long prev = atomicCAS(&hkeys[h], 0ull, key);
      if (prev == 0ull || prev == key) {
        // two value slots per key; order fixed below by segment index
        const int slot = atomicAdd(&hvals[3 * h + 2], 1);
        if (slot < 2) hvals[3 * h + slot] = e;
        else atomicOr(err, 2);  // > 2 segments on one edge (non-manifold)
        break;
      }
      h = (h + 1) & (hcap - 1);
    }
  }
}

// partner[e] = the other (segment, side) with the same key, or -1
__device__ __forceinline__ int chain_partner_of(const HydroJob& J, int e) {
  const int s = e >> 1, side = e & 1;
  const int2 k = side ? J.segs[s].kb : J.segs[s].ka;
  const unsigned long long key = key64(k) + 1ull;
  unsigned h = hash64(key) & (J.hcap - 1);
  int p = -1;
  for (int probe = 0; probe < J.hcap; ++probe) {
    if (J.hkeys[h] == key) {
      const int cnt = min(J.hvals[3 * h + 2], 2);
      for (int q = 0; q < cnt; ++q)
        if (J.hvals[3 * h + q] != e) p = J.hvals[3 * h + q];
      break;
    }
    h = (h + 1) & (J.hcap - 1);
  }
  return p;
}

// Sequential walk with the reference's visiting order (hydro.cpp:167-213) in
// shared memory. Emits point references e = 2*segment + side: the crossing
// point of that key as stored by the larger segment (std::map last writer).
constexpr int kChainSeq = 12288;  // segments of the sequential fallback in shared memory
constexpr int kChainPar = 4096;   // segments of the parallel path (2 nodes each)
constexpr int kChainThreads = 1024;

// Reference walk (hydro.cpp:167-213) by one thread: general topology
// (open chains, any size). partner / used may live in shared or global memory.
__device__ void chain_walk_seq(int nseg, const int* partner, unsigned char* used, int* loop_off,
                               int* point_ref, int* counts_out) {
  int nl = 0, np = 0;
  loop_off[0] = 0;
  auto canon = [&](int e) {
    const int p = partner[e];
    return (p >= 0 && (p >> 1) > (e >> 1)) ? p : e;
  };
  for (int start = 0; start < nseg; ++start) {
    if (used[start]) continue;
    int lp = 0, seg = start, entry = 0;
    bool closed = false;
    const int first = 2 * start;  // first_entry = start's first key
    for (;;) {
      used[seg] = 1;
      point_ref[np + lp++] = canon(2 * seg + entry);
      const int ex = 2 * seg + (1 - entry);
      const int p = partner[ex];
      if (p == first) {
        closed = true;
        break;
      }
      if (p < 0 || used[p >> 1]) {
        point_ref[np + lp++] = canon(ex);
        break;
      }
      seg = p >> 1;
      entry = p & 1;
    }
    if (lp >= 3) {
      if (closed) point_ref[np + lp] = point_ref[np], ++lp;
      np += lp;
      loop_off[++nl] = np;
    }
  }
  counts_out[0] = nl;
  counts_out[1] = np;
}

// Waterline chaining with the reference's visiting order. On a closed mesh
// every crossed edge has exactly two segments, so "segment s entered through
// side x" nodes form a permutation next(e) = partner[e ^ 1] whose cycles are
// the loops (each in both orientations). The reference walks the cycle of its
// lowest unused segment s0, entering through side 0: that is the orientation
// whose minimum node id is even (2 s0). Pointer jumping gives every node its
// cycle minimum and its distance to the start node, hence its position in the
// loop; loops are numbered by increasing s0 exactly as the reference emits
// them. Open topology (a crossed edge with one segment) or huge waterlines
// take the sequential walk.
template <int NB>
__global__ void __launch_bounds__(kChainThreads) k_chain(const __grid_constant__ HydroBatch<NB> B) {
  const HydroJob& J = B.job[blockIdx.y];
  const int2* total = J.total;
  const int* partner_g = J.partner;
  unsigned char* used_g = J.used;
  int* loop_off = J.loop_off;
  int* point_ref = J.point_ref;
  int* counts_out = J.loop_counts;
  extern __shared__ int sm_chain[];
  __shared__ int s_open;
  __shared__ int s_wsum[kChainThreads / 32];
  const int nseg = total->y;
  const int tid = threadIdx.x;
  if (tid == 0) s_open = 0;
  __syncthreads();
  const int nodes = 2 * nseg;
  for (int e = tid; e < nodes; e += blockDim.x) {  // partners from the hash table (was k_chain_partner)
    const int p = chain_partner_of(J, e);
    J.partner[e] = p;
    if (p < 0) s_open = 1;
  }
  __syncthreads();
  if (s_open || nseg > kChainPar) {
    // sequential fallback
    const bool in_smem = nseg <= kChainSeq;
    int* partner = in_smem ? sm_chain : const_cast<int*>(partner_g);
    unsigned char* used =
        in_smem ? reinterpret_cast<unsigned char*>(sm_chain + 2 * kChainSeq) : used_g;
    if (in_smem)
      for (int e = tid; e < nodes; e += blockDim.x) sm_chain[e] = partner_g[e];
    for (int q = tid; q < nseg; q += blockDim.x) used[q] = 0;
    __syncthreads();
    if (tid == 0) {
      chain_walk_seq(nseg, partner, used, loop_off, point_ref, counts_out);
      J.report->r.waterline_loops = counts_out[0];
      J.report->r.waterline_points = counts_out[1];
    }
    __syncthreads();
    const int np = counts_out[1];  // loop points (was k_chain_points)
    for (int q = tid; q < np; q += blockDim.x) {
      const int e = point_ref[q];
      const SegDev& sg = J.segs[e >> 1];
      st3(J.loop_points + 3 * q, (e & 1) ? sg.pb : sg.pa);
    }
    return;
  }
  int* prt = sm_chain;                 // [nodes] partner
  int* cmin = sm_chain + 2 * kChainPar;  // [nodes]
  int* jp = sm_chain + 4 * kChainPar;    // [nodes]
  int* dist = sm_chain + 6 * kChainPar;  // [nodes]
  int* segoff = sm_chain + 8 * kChainPar;  // [nseg] point offset of the loop starting there
  for (int e = tid; e < nodes; e += blockDim.x) {
    prt[e] = partner_g[e];
  }
  __syncthreads();
  for (int e = tid; e < nodes; e += blockDim.x) {
    cmin[e] = e;
    jp[e] = prt[e ^ 1];
  }
  __syncthreads();
  // ---- phase A: cycle minimum node id
  for (int span = 1; span < nodes; span <<= 1) {
    int nm[8], nj[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = tid + k * kChainThreads;
      if (e < nodes) {
        const int j = jp[e];
        nm[k] = min(cmin[e], cmin[j]);
        nj[k] = jp[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = tid + k * kChainThreads;
      if (e < nodes) cmin[e] = nm[k], jp[e] = nj[k];
    }
    __syncthreads();
  }
  // ---- phase B: distance to the start node (live orientation only)
  for (int e = tid; e < nodes; e += blockDim.x) {
    const int st = cmin[e];
    const bool live = (st & 1) == 0;
    dist[e] = (!live || e == st) ? 0 : 1;
    jp[e] = (!live || e == st) ? e : prt[e ^ 1];
  }
  __syncthreads();
  for (int span = 1; span < nodes; span <<= 1) {
    int nd[8], nj[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = tid + k * kChainThreads;
      if (e < nodes) {
        const int j = jp[e];
        nd[k] = dist[e] + dist[j];
        nj[k] = jp[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = tid + k * kChainThreads;
      if (e < nodes) dist[e] = nd[k], jp[e] = nj[k];
    }
    __syncthreads();
  }
  // ---- loop sizes at the start segments, exclusive scan in segment order
  // node 2 s is a start iff its cycle minimum is itself; length L = dist(next) + 1
  int keep_len[4];
  int local = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = tid * 4 + k;
    int v = 0;
    if (q < nseg) {
      const int e = 2 * q;
      if (cmin[e] == e) {
        const int L = dist[prt[e ^ 1]] + 1;
        if (L >= 3) v = L + 1;
      }
    }
    keep_len[k] = v;
    local += v;
  }
  // block exclusive scan of `local` (thread order = segment order)
  int incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((tid & 31) >= o) incl += y;
  }
  if ((tid & 31) == 31) s_wsum[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    int w = tid < kChainThreads / 32 ? s_wsum[tid] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (tid >= o) w += y;
    }
    s_wsum[tid] = w;  // inclusive warp sums
  }
  __syncthreads();
  int base = incl - local + ((tid >> 5) ? s_wsum[(tid >> 5) - 1] : 0);
  // loop numbering: count kept starts before each (second scan on 0/1 flags)
  int cnt_local = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) cnt_local += keep_len[k] > 0;
  int cincl = cnt_local;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, cincl, o);
    if ((tid & 31) >= o) cincl += y;
  }
  __shared__ int s_csum[kChainThreads / 32];
  if ((tid & 31) == 31) s_csum[tid >> 5] = cincl;
  __syncthreads();
  if (tid < 32) {
    int w = tid < kChainThreads / 32 ? s_csum[tid] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (tid >= o) w += y;
    }
    s_csum[tid] = w;
  }
  __syncthreads();
  int cbase = cincl - cnt_local + ((tid >> 5) ? s_csum[(tid >> 5) - 1] : 0);
  // segoff[q] = point offset of the loop starting at segment q (or -1)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int q = tid * 4 + k;
    if (q >= nseg) break;
    if (keep_len[k] > 0) {
      segoff[q] = base;
      loop_off[cbase + 1] = base + keep_len[k];
      ++cbase;
    } else {
      segoff[q] = -1;
    }
    base += keep_len[k];
  }
  if (tid == kChainThreads - 1) {
    counts_out[0] = s_csum[kChainThreads / 32 - 1];
    counts_out[1] = s_wsum[kChainThreads / 32 - 1];
    loop_off[0] = 0;
    J.report->r.waterline_loops = counts_out[0];  // (was k_report_loops)
    J.report->r.waterline_points = counts_out[1];
  }
  __syncthreads();
  // ---- scatter point references: position = (L - dist) mod L, closing point at L
  auto canon = [&](int e) {
    const int p = prt[e];
    return (p >= 0 && (p >> 1) > (e >> 1)) ? p : e;
  };
  for (int e = tid; e < nodes; e += blockDim.x) {
    const int st = cmin[e];
    if (st & 1) continue;  // orientation the reference never walks
    const int off = segoff[st >> 1];
    if (off < 0) continue;  // loop shorter than 3 points
    const int L = dist[prt[st ^ 1]] + 1;
    const int pos = (L - dist[e]) % L;
    const int ce = canon(e);
    const SegDev& sg = J.segs[ce >> 1];  // the point itself (was k_chain_points)
    const double3 p = (ce & 1) ? sg.pb : sg.pa;
    point_ref[off + pos] = ce;
    st3(J.loop_points + 3 * (off + pos), p);
    if (e == st) {
      point_ref[off + L] = ce;
      st3(J.loop_points + 3 * (off + L), p);
    }
  }
}




int grid_of(ocn_ctx* ctx, int n, int threads) {
  int b = (n + threads - 1) / threads;
  int cap = ctx->sm_count * 8;
  return b < 1 ? 1 : (b > cap ? cap : b);
}

}  // namespace

// ---------------------------------------------------------------- host pipeline
// The job of one mesh: pose, medium, zones and (optional) host-sampled depths;
// uploads what the evaluation reads from host memory onto the mesh's buffers.
HydroJob make_job(ocn_mesh* m, const ocn_pose* pose, const ocn_fluid* fluid,
                  const double* host_depth) {
  cudaStream_t st = m->ctx->stream;
  HydroJob J{};
  J.verts = m->verts.p, J.tris = m->tris.p, J.normals = m->normals.p, J.areas = m->areas.p;
  J.nv = m->nv, J.nt = m->nt, J.degenerate = m->degenerate, J.hcap = m->hcap;
  J.volume = m->volume;
  for (int k = 0; k < 3; ++k) {
    J.P.p[k] = pose->position[k];
    J.P.v[k] = pose->linear_velocity[k];
    J.P.w[k] = pose->angular_velocity[k];
    J.P.com[k] = pose->com_body[k];
  }
  for (int k = 0; k < 4; ++k) J.P.q[k] = pose->orientation[k];
  if (fluid && fluid->n_zones) {
    OCN_REQUIRE(fluid->n_zones <= kMaxZones, "too many zones (%d)", fluid->n_zones);
    J.zones.count = fluid->n_zones;
    for (int z = 0; z < J.zones.count; ++z) J.zones.z[z] = zone_view((ocn_zone*)fluid->zones[z]);
  }
  if (fluid) {
    for (int k = 0; k < 3; ++k) J.F.wind[k] = fluid->wind[k];
    J.F.water_density = fluid->water_density;
    J.F.air_density = fluid->air_density;
    J.F.cd_water = fluid->cd_water;
    J.F.cd_air = fluid->cd_air;
    J.F.n_profile = fluid->n_profile;
    if (fluid->n_profile > 0) {
      m->d_profile.ensure(2 * (size_t)fluid->n_profile);
      OCN_CUDA(cudaMemcpyAsync(m->d_profile.p, fluid->host_profile,
                               2 * (size_t)fluid->n_profile * sizeof(double),
                               cudaMemcpyHostToDevice, st));
      J.F.profile = m->d_profile.p;
    }
    J.clamp = fluid->velocity_clamp;
  } else {
    J.F.water_density = 1025.0;
    J.F.air_density = 1.204;
    J.F.cd_water = J.F.cd_air = 1.0;
    J.clamp = 1;
  }
  if (host_depth) {
    OCN_CUDA(cudaMemcpyAsync(m->override_depth.p, host_depth, m->nv * sizeof(double),
                             cudaMemcpyHostToDevice, st));
    J.override_depth = m->override_depth.p;
  }
  J.wpos = m->wpos.p, J.depth = m->depth.p;
  J.counts = m->counts.p, J.offsets = m->offsets.p, J.block_sums = m->block_sums.p;
  J.total = m->total.p;
  J.states = m->states.p, J.segs = m->segs.p;
  J.block_out = m->block_out.p, J.report = m->report.p, J.flags = m->flags.p;
  J.ticket = m->ticket.p;
  J.hkeys = m->hkeys.p, J.hvals = m->hvals.p, J.partner = m->partner.p, J.used = m->used.p;
  J.loop_off = m->loop_off.p, J.point_ref = m->point_ref.p, J.loop_counts = m->loop_counts.p;
  J.loop_points = m->loop_points.p;
  return J;
}

// Clip stage of every job: vertices, classification + scan, emission.
template <int NB>
void launch_clip(ocn_ctx* ctx, const HydroBatch<NB>& B, int max_nv, int max_nt) {
  cudaStream_t st = ctx->stream;
  const unsigned nb = (unsigned)B.n;
  k_vertices<NB><<<dim3(std::max(1, grid_of(ctx, 4 * max_nv, 128) / (int)nb), nb), 128, 0, st>>>(B);
  OCN_LAUNCHED(ctx);
  const int sb = (max_nt + kScanBlock - 1) / kScanBlock;
  k_classify_scan<NB><<<dim3(sb, nb), kScanBlock, 0, st>>>(B);
  OCN_LAUNCHED(ctx);
  k_emit<NB><<<dim3(std::max(1, grid_of(ctx, max_nt, 128) / (int)nb), nb), 128, 0, st>>>(B);
  OCN_LAUNCHED(ctx);
}

// Reduction and waterline stages of every job.
template <int NB>
void launch_reduce(ocn_ctx* ctx, const HydroBatch<NB>& B, int max_nt) {
  cudaStream_t st = ctx->stream;
  const unsigned nb = (unsigned)B.n;
  // the per-job partial count is fixed (block_out holds 2 sm_count partials)
  const int fblocks = std::max(8, ctx->sm_count * 2 / B.n);
  k_forces<NB><<<dim3(fblocks, nb), kForceThreads, 0, st>>>(B);
  OCN_LAUNCHED(ctx);
  const int cb = std::max(1, grid_of(ctx, 2 * max_nt, 256) / (int)nb);
  k_chain_hash<NB><<<dim3(cb, nb), 256, 0, st>>>(B);
  OCN_LAUNCHED(ctx);
  const size_t chain_smem = std::max(9 * kChainPar * sizeof(int),
                                     2 * kChainSeq * sizeof(int) + kChainSeq);
  smem_opt_in(k_chain<NB>, chain_smem);
  k_chain<NB><<<dim3(1, nb), kChainThreads, chain_smem, st>>>(B);
  OCN_LAUNCHED(ctx);
}

template <int NB>
void fill_samplers(HydroBatch<NB>& B, const ocn_fluid* fluid) {
  ocn_maps* maps = fluid ? (ocn_maps*)fluid->maps : nullptr;
  ocn_slices* slices = fluid ? (ocn_slices*)fluid->slices : nullptr;
  // maps == NULL: still water (FluidQuery::still_water, hydro.cpp:25-30) plus any zones
  B.have_surf = maps != nullptr;
  if (maps) B.surf = make_surf_view(maps);
  B.have_vel = slices != nullptr;
  if (slices) B.vel = make_slice_view(slices);
}

void hydro_evaluate(ocn_mesh* m, const ocn_pose* pose, const ocn_fluid* fluid,
                    const double* host_depth) {
  NvtxRange nv("hydro");
  ocn_ctx* ctx = m->ctx;
  DeviceScope ds(ctx);
  cudaStream_t st = ctx->stream;
  HydroBatch<1> B{};
  B.n = 1;
  fill_samplers(B, fluid);
  B.job[0] = make_job(m, pose, fluid, host_depth);
  ProfWindow pw(ctx, OCN_PROF_HYDRO);
  launch_clip(ctx, B, m->nv, m->nt);
  if (fluid && fluid->host_velocity && !fluid->slices) {
    // host water_velocity sampler (hydro.cpp:276-282): the submerged states'
    // centroids go to the host once, the callback fills their medium
    // velocities, which the force pass reads instead of velocity_at
    int2 total{};
    OCN_CUDA(cudaMemcpyAsync(&total, m->total.p, sizeof(int2), cudaMemcpyDeviceToHost, st));
    OCN_CUDA(cudaStreamSynchronize(st));
    const int ns = total.x;
    std::vector<StateDev> hs(ns);
    if (ns)
      OCN_CUDA(cudaMemcpy(hs.data(), m->states.p, ns * sizeof(StateDev), cudaMemcpyDeviceToHost));
    std::vector<double> xzy, vel;
    std::vector<int> idx;
    for (int i = 0; i < ns; ++i)
      if (hs[i].status == 0) {
        idx.push_back(i);
        xzy.insert(xzy.end(), {hs[i].centroid.x, hs[i].centroid.z, hs[i].centroid.y});
      }
    vel.assign(xzy.size(), 0.0);
    if (!idx.empty())
      fluid->host_velocity(fluid->host_velocity_user, (int64_t)idx.size(), xzy.data(), vel.data());
    m->ext_vel_host.assign(3 * (size_t)std::max(ns, 1), 0.0);
    for (size_t k = 0; k < idx.size(); ++k)
      for (int c = 0; c < 3; ++c) m->ext_vel_host[3 * (size_t)idx[k] + c] = vel[3 * k + c];
    m->ext_vel.ensure(m->ext_vel_host.size());
    OCN_CUDA(cudaMemcpyAsync(m->ext_vel.p, m->ext_vel_host.data(),
                             m->ext_vel_host.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    B.job[0].ext_vel = m->ext_vel.p;
  }
  launch_reduce(ctx, B, m->nt);
  m->evaluated = true;
}

void fill_samplers_batch(HydroBatch<kMaxBatch>& B, const ocn_fluid* fluid) {
  fill_samplers(B, fluid);
}

// Runs prepared jobs (make_job per mesh) as one launch set.
void hydro_evaluate_jobs(int n, ocn_mesh* const* meshes, const HydroBatch<kMaxBatch>& B) {
  NvtxRange nv("hydro");
  ocn_ctx* ctx = meshes[0]->ctx;
  DeviceScope ds(ctx);
  int max_nv = 0, max_nt = 0;
  for (int i = 0; i < n; ++i) {
    max_nv = std::max(max_nv, meshes[i]->nv);
    max_nt = std::max(max_nt, meshes[i]->nt);
  }
  ProfWindow pw(ctx, OCN_PROF_HYDRO);
  launch_clip(ctx, B, max_nv, max_nt);
  launch_reduce(ctx, B, max_nt);
  for (int i = 0; i < n; ++i) meshes[i]->evaluated = true;
}

// Simulation::step's body loop (sim.cpp:74-83) as one launch set: job i is
// meshes[i] at poses[i] against fluids[i] (its own zones / drag constants, zone
// views taken now); every fluid shares the maps and slices.
void hydro_evaluate_batch(int n, ocn_mesh* const* meshes, const ocn_pose* poses,
                          const ocn_fluid* fluids) {
  ocn_ctx* ctx = meshes[0]->ctx;
  DeviceScope ds(ctx);
  HydroBatch<kMaxBatch> B{};
  B.n = n;
  fill_samplers(B, &fluids[0]);
  for (int i = 0; i < n; ++i) {
    OCN_REQUIRE(meshes[i] && meshes[i]->ctx == ctx, "batched meshes must share one context");
    OCN_REQUIRE(fluids[i].maps == fluids[0].maps && fluids[i].slices == fluids[0].slices,
                "batched evaluations must share the surface and velocity samplers");
    OCN_REQUIRE(!fluids[i].host_velocity || fluids[i].slices,
                "host velocity samplers are not batched (use ocn_hydro_aggregate)");
    B.job[i] = make_job(meshes[i], &poses[i], &fluids[i], nullptr);
  }
  hydro_evaluate_jobs(n, meshes, B);
}

void hydro_check_flags(ocn_mesh* m) {
  int flags[4];
  OCN_CUDA(cudaMemcpy(flags, m->flags.p, sizeof(flags), cudaMemcpyDeviceToHost));
  if (flags[0]) fail(OCN_ERR_DOMAIN, "velocity_at: depth outside [y_min, y_max]");
  if (flags[1]) fail(OCN_ERR_MESH, "waterline: an edge is shared by more than two triangles");
}

// The reports (and error flags) of n evaluated meshes on one context: async
// copies into each mesh's pinned staging, one stream synchronisation.
void hydro_reports_read(int n, ocn_mesh* const* meshes, ocn_hydro_report* out) {
  if (n <= 0) return;
  ocn_ctx* ctx = meshes[0]->ctx;
  DeviceScope ds(ctx);
  for (int i = 0; i < n; ++i) {
    ocn_mesh* m = meshes[i];
    OCN_REQUIRE(m && m->ctx == ctx, "meshes of one context");
    OCN_REQUIRE(m->evaluated, "no hydro evaluation yet");
    if (!m->h_report) {
      OCN_CUDA(cudaMallocHost(&m->h_report, sizeof(ReportDev)));
      OCN_CUDA(cudaMallocHost(&m->h_flags, 4 * sizeof(int)));
    }
    OCN_CUDA(cudaMemcpyAsync(m->h_report, m->report.p, sizeof(ReportDev), cudaMemcpyDeviceToHost,
                             ctx->stream));
    OCN_CUDA(cudaMemcpyAsync(m->h_flags, m->flags.p, 4 * sizeof(int), cudaMemcpyDeviceToHost,
                             ctx->stream));
  }
  OCN_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n; ++i) {
    const ocn_mesh* m = meshes[i];
    if (m->h_flags[0]) fail(OCN_ERR_DOMAIN, "velocity_at: depth outside [y_min, y_max]");
    if (m->h_flags[1]) fail(OCN_ERR_MESH, "waterline: an edge is shared by more than two triangles");
    out[i] = m->h_report->r;
  }
}

}  // namespace ocn

using namespace ocn;

extern "C" {

int ocn_mesh_create(ocn_ctx* ctx, int nv, const double* verts, int nt, const int32_t* tris,
                    const double* normals, const double* areas, double volume, ocn_mesh** out) {
  return api_call(ctx, [&] {
    OCN_REQUIRE(ctx && out && verts && tris && normals && areas, "null argument");
    if (nv <= 0 || nt <= 0) fail(OCN_ERR_MESH, "empty mesh");
    DeviceScope ds(ctx);
    auto m = std::make_unique<ocn_mesh>();
    m->ctx = ctx;
    m->nv = nv;
    m->nt = nt;
    m->volume = volume;
    for (int t = 0; t < nt; ++t) {
      for (int k = 0; k < 3; ++k)
        if (tris[3 * t + k] < 0 || tris[3 * t + k] >= nv)
          fail(OCN_ERR_MESH, "mesh: face references a missing vertex");
      if (areas[t] <= 0.0) ++m->degenerate;
    }
    m->verts.alloc(3 * (size_t)nv);
    m->tris.alloc(nt);
    m->normals.alloc(3 * (size_t)nt);
    m->areas.alloc(nt);
    OCN_CUDA(cudaMemcpy(m->verts.p, verts, 3 * (size_t)nv * sizeof(double), cudaMemcpyHostToDevice));
    OCN_CUDA(cudaMemcpy(m->tris.p, tris, (size_t)nt * sizeof(int3), cudaMemcpyHostToDevice));
    OCN_CUDA(cudaMemcpy(m->normals.p, normals, 3 * (size_t)nt * sizeof(double), cudaMemcpyHostToDevice));
    OCN_CUDA(cudaMemcpy(m->areas.p, areas, (size_t)nt * sizeof(double), cudaMemcpyHostToDevice));
    m->wpos.alloc(3 * (size_t)nv);
    m->depth.alloc(nv);
    m->override_depth.alloc(nv);
    m->counts.alloc(nt);
    m->offsets.alloc(nt);
    m->block_sums.alloc((nt + kScanBlock - 1) / kScanBlock + 1);
    m->total.alloc(1);
    m->states.alloc(3 * (size_t)nt);
    m->segs.alloc(nt);
    m->block_out.alloc((size_t)ctx->sm_count * 2 * kTerms);
    m->report.alloc(1);
    m->flags.alloc(4);
    m->ticket.alloc(1);
    OCN_CUDA(cudaMemset(m->ticket.p, 0, sizeof(int)));
    int hcap = 1;
    while (hcap < 4 * nt) hcap <<= 1;
    m->hcap = hcap;
    m->hkeys.alloc(hcap);
    m->hvals.alloc(3 * (size_t)hcap);
    m->partner.alloc(2 * (size_t)nt);
    m->used.alloc(nt);
    m->loop_off.alloc((size_t)nt + 2);
    m->point_ref.alloc(2 * (size_t)nt + 2);
    m->loop_points.alloc(3 * (2 * (size_t)nt + 2));
    m->loop_counts.alloc(2);
    OCN_CUDA(cudaMemset(m->total.p, 0, sizeof(int2)));
    OCN_CUDA(cudaMemset(m->loop_counts.p, 0, 2 * sizeof(int)));
    ctx_retain(ctx);
    *out = m.release();
  });
}

int ocn_mesh_destroy(ocn_mesh* m) {
  if (!m) return OCN_OK;
  ocn_ctx* ctx = m->ctx;
  {
    DeviceScope ds(ctx);
    cudaStreamSynchronize(ctx->stream);
    delete m;
  }
  ctx_release(ctx);
  return OCN_OK;
}

int ocn_hydro_aggregate(ocn_mesh* m, const ocn_pose* pose, const ocn_fluid* fluid,
                        const double* host_depth, ocn_hydro_report* report) {
  return api_call(m ? m->ctx : nullptr, [&] {
    OCN_REQUIRE(m && pose, "null argument");
    hydro_evaluate(m, pose, fluid, host_depth);
    if (report) {
      ReportDev r;
      OCN_CUDA(cudaMemcpyAsync(&r, m->report.p, sizeof(r), cudaMemcpyDeviceToHost, m->ctx->stream));
      OCN_CUDA(cudaStreamSynchronize(m->ctx->stream));
      hydro_check_flags(m);
      *report = r.r;
    }
  });
}

int ocn_hydro_aggregate_batch(int n, ocn_mesh* const* meshes, const ocn_pose* poses,
                              const ocn_fluid* fluids, ocn_hydro_report* reports) {
  ocn_ctx* ctx = n > 0 && meshes && meshes[0] ? meshes[0]->ctx : nullptr;
  return api_call(ctx, [&] {
    OCN_REQUIRE(n >= 0 && n <= kMaxBatch, "batch of %d meshes (1..%d)", n, kMaxBatch);
    if (n == 0) return;
    OCN_REQUIRE(meshes && poses && fluids, "null argument");
    hydro_evaluate_batch(n, meshes, poses, fluids);
    if (reports) hydro_reports_read(n, meshes, reports);
  });
}

int ocn_hydro_report_get(ocn_mesh* m, ocn_hydro_report* report) {
  return api_call(m ? m->ctx : nullptr, [&] {
    OCN_REQUIRE(m && report, "null argument");
    hydro_reports_read(1, &m, report);
  });
}

int ocn_hydro_reports_get(int n, ocn_mesh* const* meshes, ocn_hydro_report* reports) {
  return api_call(n > 0 && meshes && meshes[0] ? meshes[0]->ctx : nullptr, [&] {
    OCN_REQUIRE(n >= 0 && (n == 0 || (meshes && reports)), "null argument");
    hydro_reports_read(n, meshes, reports);
  });
}

int ocn_hydro_vertices(ocn_mesh* m, double* world, double* depth) {
  return api_call(m ? m->ctx : nullptr, [&] {
    OCN_REQUIRE(m && m->evaluated, "no hydro evaluation yet");
    DeviceScope ds(m->ctx);
    OCN_CUDA(cudaStreamSynchronize(m->ctx->stream));
    if (world)
      OCN_CUDA(cudaMemcpy(world, m->wpos.p, 3 * (size_t)m->nv * sizeof(double), cudaMemcpyDeviceToHost));
    if (depth)
      OCN_CUDA(cudaMemcpy(depth, m->depth.p, (size_t)m->nv * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int ocn_hydro_states(ocn_mesh* m, int capacity, ocn_triangle_state* out, int* count) {
  return api_call(m ? m->ctx : nullptr, [&] {
    OCN_REQUIRE(m && m->evaluated, "no hydro evaluation yet");
    DeviceScope ds(m->ctx);
    OCN_CUDA(cudaStreamSynchronize(m->ctx->stream));
    int2 tot;
    OCN_CUDA(cudaMemcpy(&tot, m->total.p, sizeof(tot), cudaMemcpyDeviceToHost));
    if (count) *count = tot.x;
    if (out && capacity > 0) {
      int n = std::min(capacity, tot.x);
      std::vector<StateDev> tmp(n);
      OCN_CUDA(cudaMemcpy(tmp.data(), m->states.p, n * sizeof(StateDev), cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) {
        out[i].parent = tmp[i].parent;
        out[i].status = tmp[i].status;
        out[i].area = tmp[i].area;
        out[i].centroid[0] = tmp[i].centroid.x;
        out[i].centroid[1] = tmp[i].centroid.y;
        out[i].centroid[2] = tmp[i].centroid.z;
        out[i].depth = tmp[i].depth;
        out[i].normal[0] = tmp[i].normal.x;
        out[i].normal[1] = tmp[i].normal.y;
        out[i].normal[2] = tmp[i].normal.z;
      }
    }
  });
}

int ocn_hydro_waterline(ocn_mesh* m, int* n_loops, int* n_points, int32_t* offsets, double* points) {
  return api_call(m ? m->ctx : nullptr, [&] {
    OCN_REQUIRE(m && m->evaluated, "no hydro evaluation yet");
    DeviceScope ds(m->ctx);
    OCN_CUDA(cudaStreamSynchronize(m->ctx->stream));
    int cnt[2];
    OCN_CUDA(cudaMemcpy(cnt, m->loop_counts.p, sizeof(cnt), cudaMemcpyDeviceToHost));
    if (n_loops) *n_loops = cnt[0];
    if (n_points) *n_points = cnt[1];
    if (offsets)
      OCN_CUDA(cudaMemcpy(offsets, m->loop_off.p, (cnt[0] + 1) * sizeof(int), cudaMemcpyDeviceToHost));
    if (points && cnt[1] > 0)
      OCN_CUDA(cudaMemcpy(points, m->loop_points.p, 3 * (size_t)cnt[1] * sizeof(double),
                          cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
