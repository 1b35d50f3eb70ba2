// K3/K4/K7 — pair forces over full Verlet lists, energy/virial reduction, and
// the fused production timestep kernel (reference: compute_forces,
// potential.py:134-213; laws potential.py:30-97; integrators driver.py:74-93).
//
// Layout: positions/velocities/forces SoA fp64 with leading
// dimension ld; lists int32 neighbor-major.  One thread owns one local atom:
// its accumulation is a private register sum (no atomics, no shared writes),
// the list slot k of 32 consecutive atoms is one coalesced 128-byte load, and
// the x_j gathers of a warp hit a handful of L1/L2 lines because list slots of
// neighbouring atoms point at neighbouring cells.
//
// Two LJ kernels:
//  * EXACT  — the reference's operation order with explicit round-to-nearest
//             ops and sequential list-order accumulation: bitwise equal to
//             compute_forces on the same lists.
//  * fast   — FMA-contracted rsq/accumulation and a Newton-refined hardware
//             reciprocal instead of IEEE division (rel. error ~1e-14, far
//             inside the 1e-10 parity bound).
//
// The production step kernels (k_step, tmd_step_lj / tmd_step_sd) run
// 256-atom blocks at 4 per SM (64 registers); between two list rebuilds their
// launches are issued by tmd_run_steps (bottom of this file), one host call.
#include "tmd_common.cuh"

namespace tmd {

// ---------------------------------------------------------------------------
// pair laws in reference order (potential.py:46-57, 80-97)
// ---------------------------------------------------------------------------
struct LJExact {
  double eps, sigma6;
  // f = (((48 sr6) (sr6 - 0.5)) sr2) eps, sr6 = ((sr2 sr2) sr2) sigma6, sr2 = 1 / rsq
  __device__ __forceinline__ double scalar(double rsq) const {
    double sr2 = div_rn(1.0, rsq);
    double sr6 = mul_rn(mul_rn(mul_rn(sr2, sr2), sr2), sigma6);
    return mul_rn(mul_rn(mul_rn(mul_rn(48.0, sr6), sub_rn(sr6, 0.5)), sr2), eps);
  }
  // 4 eps (sr6^2 - sr6), sr6 = sigma6 / rsq^3
  __device__ __forceinline__ double energy(double rsq) const {
    double sr6 = div_rn(sigma6, mul_rn(mul_rn(rsq, rsq), rsq));
    return mul_rn(mul_rn(4.0, eps), sub_rn(mul_rn(sr6, sr6), sr6));
  }
};

struct SDExact {
  double k, gamma, diam;
  // returns contact flag; out = K ov n - gamma (n.(vi - vj)) n
  __device__ __forceinline__ bool force(double dx, double dy, double dz, double rsq, double vix,
                                        double viy, double viz, double vjx, double vjy, double vjz,
                                        double& fx, double& fy, double& fz) const {
    double dist = __dsqrt_rn(rsq);
    double ov = sub_rn(diam, dist);
    if (!(ov > 0.0)) {
      fx = fy = fz = 0.0;
      return false;
    }
    double ux = div_rn(dx, dist), uy = div_rn(dy, dist), uz = div_rn(dz, dist);
    double ko = mul_rn(k, ov);
    double rx = sub_rn(vix, vjx), ry = sub_rn(viy, vjy), rz = sub_rn(viz, vjz);
    double vn = add_rn(add_rn(mul_rn(ux, rx), mul_rn(uz, rz)), mul_rn(uy, ry));
    double gv = mul_rn(-gamma, vn);
    fx = add_rn(mul_rn(ko, ux), mul_rn(gv, ux));
    fy = add_rn(mul_rn(ko, uy), mul_rn(gv, uy));
    fz = add_rn(mul_rn(ko, uz), mul_rn(gv, uz));
    return true;
  }
  __device__ __forceinline__ double energy(double rsq) const {
    double ov = fmax(sub_rn(diam, __dsqrt_rn(rsq)), 0.0);
    return mul_rn(mul_rn(mul_rn(0.5, k), ov), ov);
  }
};

__device__ __forceinline__ void report_singular(int64_t* st, int32_t i, int32_t k) {
  raise_status(st, TMD_SINGULARITY, ((unsigned long long)(uint32_t)i << 32) | (uint32_t)k);
}

// ---------------------------------------------------------------------------
// exact LJ: bitwise equal to the reference on the same lists
// ---------------------------------------------------------------------------
template <bool ENERGY>
__global__ void __launch_bounds__(128) k_force_lj_exact(
    const double* __restrict__ pos, int64_t ld, int32_t n, const int32_t* __restrict__ nbr,
    int64_t ld_nbr, const int32_t* __restrict__ nnbr, int32_t cap, double rc2, LJExact law,
    double* __restrict__ frc, int64_t ld_f, double* partials, unsigned int* counter,
    double* thermo, int64_t* st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double red[2] = {0.0, 0.0};
  if (i < n) {
    const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
    const int32_t cnt = nnbr[i];
    double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0, w = 0.0;
    for (int32_t k = 0; k < cnt; ++k) {
      const int32_t j = nbr[slot_index(k, i, ld_nbr)];
      const double dx = sub_rn(xi, pos[j]);
      const double dy = sub_rn(yi, pos[ld + j]);
      const double dz = sub_rn(zi, pos[2 * ld + j]);
      const double rsq = rsq_ref(dx, dy, dz);
      double px = 0.0, py = 0.0, pz = 0.0;
      if (rsq < rc2) {
        if (rsq == 0.0) report_singular(st, i, k);
        const double f = law.scalar(rsq);
        px = mul_rn(f, dx);
        py = mul_rn(f, dy);
        pz = mul_rn(f, dz);
        if (ENERGY) {
          e += law.energy(rsq);
          w += px * dx + py * dy + pz * dz;
        }
      }
      // potential.py:185 sums the slots left to right starting from slot 0
      if (k == 0) {
        fx = px; fy = py; fz = pz;
      } else {
        fx = add_rn(fx, px); fy = add_rn(fy, py); fz = add_rn(fz, pz);
      }
    }
    if (cnt < cap) {  // padded slots contribute +0.0 (matters only for -0.0)
      fx = add_rn(fx, 0.0); fy = add_rn(fy, 0.0); fz = add_rn(fz, 0.0);
    }
    frc[i] = fx;
    frc[ld_f + i] = fy;
    frc[2 * ld_f + i] = fz;
    red[0] = e;
    red[1] = w;
  }
  if (ENERGY) {
    __shared__ double sm[64];
    block_sum<2>(red, sm);
    double v[2] = {0.5 * red[0], 0.5 * red[1]};
    grid_sum_finish<2>(v, partials, counter, thermo, false);
  }
}

// ---------------------------------------------------------------------------
// fast LJ body shared by the force-only kernel and the fused step kernel
//
// Software pipeline per thread: the int4 holding candidates 4q..4q+3 is
// fetched two quads ahead, bypassing L1 (the list is streamed once; L1 keeps
// the reused neighbour positions), and the 12 position gathers of a quad are
// issued together before any of the quad's arithmetic.
//
// Arithmetic per candidate (18 FP64 operations): 3 DADD (delta), 3 (rsq, FMA
// contracted), the cutoff compare, the reciprocal as the MUFU.RCP64H seed
// plus one Newton step with the cubic correction r (1 + e + e^2) (3 DFMA;
// max relative error 2.2e-16, measured over 5e6 arguments), the force
// magnitude with the constants folded, f = (A t - B) t sr2 with t = sr2^3,
// A = 48 eps sigma^12, B = 24 eps sigma^6 (5 ops), and 3 DFMA to accumulate.
// The reference computes f = (((48 sr6) (sr6 - 0.5)) sr2) eps with
// sr6 = sr2^3 sigma^6 (potential.py:46-52): the same value up to rounding.
// ---------------------------------------------------------------------------
struct LJFast {
  double rc2;
  double A, B;  // force:  f = (A t - B) t sr2
  double C, D;  // energy: e = (C t - D) t   (4 eps (sr6^2 - sr6))
};

inline LJFast lj_fast_params(double rc2, double eps, double sigma6) {
  return LJFast{rc2, 48.0 * eps * sigma6 * sigma6, 24.0 * eps * sigma6, 4.0 * eps * sigma6 * sigma6,
                4.0 * eps * sigma6};
}

// seed + one Newton step with cubic correction: r (1 + e + e^2), e = 1 - x r
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// list quads are read once per step: no L1 allocation
__device__ __forceinline__ int4 ld_quad(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Exact pruning with split rows: the production lists hold the "near" pairs
// (r_build < rc + m) at the front of each row and the rest at the back.  With
// d_i = |x_i - x_i,ref| and d = the largest displacement of any atom visible
// here (locals and ghosts; the previous step's fused epilogue leaves its
// square on the device), a back-segment pair is now farther than
// rc + m - d_i - d; while d_i + d <= m - 1e-9 the back segment is skipped.
// Forces are then identical to scanning the whole row.
struct Prune {
  const int32_t* nnear;  // near count per atom; null = single-segment rows (nnbr)
  const double* disp2;   // max squared displacement since the build
  double lim;            // m - 1e-9 (< 0: never prune)
  int32_t cap4;          // row width in slots (multiple of 4)
};

struct RowSegs {
  int32_t front, back;  // entries at [0, front) and [cap4 - back, cap4)
};

// nn / nb: the atom's near and total counts (nn = nb for single-segment rows);
// di2: its squared displacement since the build (unused without pruning)
__device__ __forceinline__ RowSegs row_segments(int32_t nn, int32_t nb, const Prune& pr, double di2) {
  if (pr.nnear == nullptr) return RowSegs{nb, 0};
  const bool skip = sqrt(di2) + sqrt(*pr.disp2) <= pr.lim;
  return RowSegs{nn, skip ? 0 : nb - nn};
}

// One contiguous run of quads [q0, q0 + nq) of atom i's row; FRONT runs mask
// slots >= hi, back runs slots < lo.  No per-candidate singularity test: a
// coincident pair within rc makes the reciprocal (and so the force)
// non-finite, which the caller checks once per atom.
// `pre` (front runs from q0 = 0 only): the first two quads were loaded by the
// caller at the start of the kernel, before the per-atom bookkeeping, so the
// row's first DRAM round trip overlaps it (the row has at least two quads;
// quads past the count are masked and never gathered from).
template <bool ENERGY, bool FRONT>
__device__ __forceinline__ void lj_segment(const double* __restrict__ pos, int64_t ld, int32_t i, double xi,
                                           double yi, double zi, const int4* __restrict__ row, int64_t ld_nbr,
                                           int32_t q0, int32_t nq, int32_t lo, int32_t hi, const LJFast& p,
                                           double& fx, double& fy, double& fz, double& e, double& w,
                                           const int4* pre = nullptr) {
  const double* __restrict__ py_ = pos + ld;
  const double* __restrict__ pz_ = pos + 2 * ld;
  const int4 self4 = make_int4(i, i, i, i);
  int4 a = pre ? pre[0] : (nq > 0 ? ld_quad(row + (int64_t)q0 * ld_nbr) : self4);
  int4 b = pre ? pre[1] : (nq > 1 ? ld_quad(row + (int64_t)(q0 + 1) * ld_nbr) : self4);
  for (int32_t v = 0; v < nq; ++v) {
    const int4 c = (v + 2 < nq) ? ld_quad(row + (int64_t)(q0 + v + 2) * ld_nbr) : self4;
    const int32_t jj[4] = {a.x, a.y, a.z, a.w};
    const int32_t s0 = 4 * (q0 + v);
    double xj[4], yj[4], zj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      xj[u] = __ldg(pos + jj[u]);
      yj[u] = __ldg(py_ + jj[u]);
      zj[u] = __ldg(pz_ + jj[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double dx = xi - xj[u];
      const double dy = yi - yj[u];
      const double dz = zi - zj[u];
      const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
      // branch-free: inside a scanned segment nearly every candidate is within
      // rc, so predicated arithmetic on a safe argument beats a divergent branch
      const bool in = (FRONT ? (s0 + u < hi) : (s0 + u >= lo)) && rsq < p.rc2;
      const double sr2 = rcp_fast(in ? rsq : 1.0);
      const double t = sr2 * sr2 * sr2;
      const double f = in ? fma(p.A, t, -p.B) * (t * sr2) : 0.0;
      fx = fma(f, dx, fx);
      fy = fma(f, dy, fy);
      fz = fma(f, dz, fz);
      if (ENERGY) {
        e = in ? fma(fma(p.C, t, -p.D), t, e) : e;
        w = fma(f, rsq, w);
      }
    }
    a = b;
    b = c;
  }
}

// Spring-Dashpot (potential.py:60-97), production arithmetic: with
// inv = 1/|delta| (MUFU.RSQ64H seed + one second-order correction, 5 DFMA),
// dist = rsq inv, overlap = d - dist, vn = (delta . (v_i - v_j)) inv,
// F = (K overlap - gamma vn) inv delta while rsq < d^2 and overlap > 0 --
// the reference's K overlap n - gamma (n . dv) n with n = delta / dist.
struct SDFast {
  double d2, diam, k, gamma, halfk;
};

__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = fma(-x * y, y, 1.0);  // 1 - x y^2
  return fma(y, h * fma(0.375, h, 0.5), y);
}

template <bool ENERGY, bool FRONT>
__device__ __forceinline__ void sd_segment(const double* __restrict__ pos, const double* __restrict__ vel, int64_t ld,
                                           int32_t i, double xi, double yi, double zi, double vxi, double vyi,
                                           double vzi, const int4* __restrict__ row, int64_t ld_nbr, int32_t q0,
                                           int32_t nq, int32_t lo, int32_t hi, const SDFast& p, double& fx,
                                           double& fy, double& fz, double& e, double& w,
                                           const int4* pre = nullptr) {
  const int4 self4 = make_int4(i, i, i, i);
  int4 a = pre ? pre[0] : (nq > 0 ? ld_quad(row + (int64_t)q0 * ld_nbr) : self4);
  for (int32_t v = 0; v < nq; ++v) {
    const int4 nx = (v + 1 < nq) ? ld_quad(row + (int64_t)(q0 + v + 1) * ld_nbr) : self4;
    const int32_t jj[4] = {a.x, a.y, a.z, a.w};
    const int32_t s0 = 4 * (q0 + v);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two candidates at a time: 12 gathers in flight
      double xj[2], yj[2], zj[2], uj[2], vj[2], wj[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int32_t j = jj[2 * h + u];
        xj[u] = __ldg(pos + j);
        yj[u] = __ldg(pos + ld + j);
        zj[u] = __ldg(pos + 2 * ld + j);
        uj[u] = __ldg(vel + j);
        vj[u] = __ldg(vel + ld + j);
        wj[u] = __ldg(vel + 2 * ld + j);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int32_t slot = s0 + 2 * h + u;
        const double dx = xi - xj[u], dy = yi - yj[u], dz = zi - zj[u];
        const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
        const bool cand = (FRONT ? (slot < hi) : (slot >= lo)) && rsq < p.d2;
        const double inv = rsqrt_fast(cand ? rsq : 1.0);
        const double ov = p.diam - rsq * inv;
        const bool in = cand && ov > 0.0;
        const double vn = fma(dx, vxi - uj[u], fma(dy, vyi - vj[u], dz * (vzi - wj[u]))) * inv;
        const double sc = in ? fma(p.k, ov, -p.gamma * vn) * inv : 0.0;
        fx = fma(sc, dx, fx);
        fy = fma(sc, dy, fy);
        fz = fma(sc, dz, fz);
        if (ENERGY) {
          e = in ? fma(p.halfk * ov, ov, e) : e;
          w = fma(sc, rsq, w);
        }
      }
    }
    a = nx;
  }
}

// Error path only: the first slot of atom i's scanned segments holding a
// partner at zero distance within rc (the segment end if none: a non-finite
// input rather than a coincident pair).
__device__ __noinline__ int32_t find_singular(const double* __restrict__ pos, int64_t ld, int32_t i,
                                              const int32_t* __restrict__ nbr, int64_t ld_nbr, RowSegs sg,
                                              int32_t cap4, double rc2) {
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int32_t end = sg.back > 0 ? cap4 : sg.front;
  for (int32_t k = 0; k < end; ++k) {
    if (!(k < sg.front || k >= cap4 - sg.back)) continue;
    const int32_t j = nbr[slot_index(k, i, ld_nbr)];
    const double dx = xi - pos[j], dy = yi - pos[ld + j], dz = zi - pos[2 * ld + j];
    const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
    if (rsq == 0.0 && rsq < rc2) return k;
  }
  return end;
}

template <bool ENERGY>
__device__ __forceinline__ void lj_fast_atom(const double* __restrict__ pos, int64_t ld, int32_t i, double xi,
                                             double yi, double zi, const int32_t* __restrict__ nbr, int64_t ld_nbr,
                                             RowSegs sg, int32_t cap4, const LJFast& p, double& fx, double& fy,
                                             double& fz, double& e, double& w, int64_t* st,
                                             const int4* pre = nullptr) {
  const int4* __restrict__ row = reinterpret_cast<const int4*>(nbr) + i;
  fx = fy = fz = e = w = 0.0;
  lj_segment<ENERGY, true>(pos, ld, i, xi, yi, zi, row, ld_nbr, 0, (sg.front + 3) >> 2, 0, sg.front, p, fx, fy, fz,
                           e, w, pre);
  if (sg.back > 0) {
    const int32_t qb = (sg.back + 3) >> 2;
    lj_segment<ENERGY, false>(pos, ld, i, xi, yi, zi, row, ld_nbr, (cap4 >> 2) - qb, qb, cap4 - sg.back, cap4, p,
                              fx, fy, fz, e, w);
  }
  if (!isfinite(fx + fy + fz)) report_singular(st, i, find_singular(pos, ld, i, nbr, ld_nbr, sg, cap4, p.rc2));
}

template <bool ENERGY>
__device__ __forceinline__ void sd_fast_atom(const double* __restrict__ pos, const double* __restrict__ vel,
                                             int64_t ld, int32_t i, double xi, double yi, double zi,
                                             const int32_t* __restrict__ nbr, int64_t ld_nbr, RowSegs sg, int32_t cap4,
                                             const SDFast& p, double& fx, double& fy, double& fz, double& e,
                                             double& w, int64_t* st, const int4* pre = nullptr) {
  const int4* __restrict__ row = reinterpret_cast<const int4*>(nbr) + i;
  const double vxi = vel[i], vyi = vel[ld + i], vzi = vel[2 * ld + i];
  fx = fy = fz = e = w = 0.0;
  sd_segment<ENERGY, true>(pos, vel, ld, i, xi, yi, zi, vxi, vyi, vzi, row, ld_nbr, 0, (sg.front + 3) >> 2, 0,
                           sg.front, p, fx, fy, fz, e, w, pre);
  if (sg.back > 0) {
    const int32_t qb = (sg.back + 3) >> 2;
    sd_segment<ENERGY, false>(pos, vel, ld, i, xi, yi, zi, vxi, vyi, vzi, row, ld_nbr, (cap4 >> 2) - qb, qb,
                              cap4 - sg.back, cap4, p, fx, fy, fz, e, w);
  }
  if (!isfinite(fx + fy + fz)) report_singular(st, i, find_singular(pos, ld, i, nbr, ld_nbr, sg, cap4, p.d2));
}

// Launch shape of the fast LJ kernels: 256-atom blocks, 3 per SM (80
// registers) for the forces-only kernel, 4 per SM for the step kernels (below).  Measured on the thermalised 80^3 lattice: forces only, front
// segments, 128 x 8 blocks (64 registers) 0.354 ms, 128 x 6 0.330, 256 x 3
// 0.323, 512 x 2 0.347 -- fewer, spatially compact blocks keep more of their
// neighbours' positions in L1.  The fused step kernel must still fit 80
// registers with a quad's 12 gathers issued together: with its per-atom loads
// issued up front (below) it does, and 3 blocks per SM beat 2 (128
// registers) by 10% (A/B on one box, scripts/gpu_ab.sh: 0.374 vs 0.413 ms);
// the LJ step at 4 blocks per SM (64 registers, no spills) beats 3 by 3%
// (0.359 vs 0.371 ms); the Spring-Dashpot step too, despite a 72-byte spill
// (C5: 0.0350 vs 0.0359 ms).
constexpr int kLJBlock = 256;
constexpr int kLJMinBlocks = 3;
#ifndef TMD_STEP_BLOCK
#define TMD_STEP_BLOCK 256
#endif
constexpr int kStepBlock = TMD_STEP_BLOCK;
constexpr int kStepMinBlocksLJ = 1024 / kStepBlock;
constexpr int kStepMinBlocksSD = 1024 / kStepBlock;

template <bool ENERGY>
__global__ void __launch_bounds__(kLJBlock, kLJMinBlocks) k_force_lj_fast(
    const double* __restrict__ pos, int64_t ld, int32_t n, const int32_t* __restrict__ nbr,
    int64_t ld_nbr, const int32_t* __restrict__ nnbr, LJFast p, double* __restrict__ frc,
    int64_t ld_f, double* partials, unsigned int* counter, double* thermo, int64_t* st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double red[2] = {0.0, 0.0};
  if (i < n) {
    double fx, fy, fz, e, w;
    lj_fast_atom<ENERGY>(pos, ld, i, pos[i], pos[ld + i], pos[2 * ld + i], nbr, ld_nbr, RowSegs{nnbr[i], 0}, 0, p,
                         fx, fy, fz, e, w, st);
    frc[i] = fx;
    frc[ld_f + i] = fy;
    frc[2 * ld_f + i] = fz;
    red[0] = e;
    red[1] = w;
  }
  if (ENERGY) {
    __shared__ double sm[64];
    block_sum<2>(red, sm);
    double v[2] = {0.5 * red[0], 0.5 * red[1]};
    grid_sum_finish<2>(v, partials, counter, thermo, false);
  }
}

// ---------------------------------------------------------------------------
// fused timestep: forces(k) -> final kick(k) [-> thermo(k)] -> kick+drift(k+1)
// ---------------------------------------------------------------------------
// Per-atom tail of the fused step: [store F], final kick, thermo terms, next
// kick + drift into pos_out, fused ghost refresh, guard displacement.
// Per-atom streams (velocities, x_ref, counts) are read and written once per
// step: streaming (evict-first) accesses keep L1 for the neighbour positions.
template <bool ENERGY>
__device__ __forceinline__ void step_atom_tail(int32_t i, double xi, double yi, double zi, double fx, double fy,
                                               double fz, double e, double w, double* __restrict__ pos_out,
                                               const double* vel, double* vel_out, int64_t ld, const Exports& ex,
                                               double c, double dt, int phases, bool store_f,
                                               double* __restrict__ frc, int64_t ld_f, bool guard, double xr,
                                               double yr, double zr, double (&red)[6], double& d2) {
  if (store_f) {
    __stcs(frc + i, fx);
    __stcs(frc + ld_f + i, fy);
    __stcs(frc + 2 * ld_f + i, fz);
  }
  // final_integrate (driver.py:86-93): v += c F, reference rounding
  double vx = __ldcs(vel + i), vy = __ldcs(vel + ld + i), vz = __ldcs(vel + 2 * ld + i);
  if (phases & TMD_PHASE_FINAL) {
    vx = add_rn(vx, mul_rn(c, fx));
    vy = add_rn(vy, mul_rn(c, fy));
    vz = add_rn(vz, mul_rn(c, fz));
  }
  if (ENERGY) {
    red[0] += e;
    red[1] += w;
    red[2] += vx * vx + vy * vy + vz * vz;
    red[3] += vx;
    red[4] += vy;
    red[5] += vz;
  }
  if (phases & TMD_PHASE_NEXT) {
    // initial_integrate of the next step (driver.py:74-83)
    vx = add_rn(vx, mul_rn(c, fx));
    vy = add_rn(vy, mul_rn(c, fy));
    vz = add_rn(vz, mul_rn(c, fz));
    const double x = add_rn(xi, mul_rn(dt, vx));
    const double y = add_rn(yi, mul_rn(dt, vy));
    const double z = add_rn(zi, mul_rn(dt, vz));
    // drift into the other position buffer: blocks still running read pos
    __stcs(pos_out + i, x);
    __stcs(pos_out + ld + i, y);
    __stcs(pos_out + 2 * ld + i, z);
    write_exports_at(ex, i, x, y, z, xr, yr, zr);
    if (guard) d2 = fmax(d2, norm2_seq(sub_rn(x, xr), sub_rn(y, yr), sub_rn(z, zr)));
  }
  __stcs(vel_out + i, vx);
  __stcs(vel_out + ld + i, vy);
  __stcs(vel_out + 2 * ld + i, vz);
}

template <bool ENERGY>
__device__ __forceinline__ void step_block_finish(int phases, const double* xref, double d2, double* dispmax2,
                                                  double (&red)[6], double* partials, unsigned int* counter,
                                                  double* thermo) {
  if ((phases & TMD_PHASE_NEXT) && xref) {
    // one atomic per block (a same-address atomic per warp serialises ~64k
    // operations per step at 2M atoms)
    __shared__ double wmax[32];
    const double m = warp_max(d2);
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      const double v = warp_max(threadIdx.x < (blockDim.x >> 5) ? wmax[threadIdx.x] : 0.0);
      if (threadIdx.x == 0) atomic_max_nonneg(dispmax2, v);
    }
  }
  if (ENERGY) {
    __shared__ double sm[6 * 32];
    block_sum<6>(red, sm);
    double v[6] = {0.5 * red[0], 0.5 * red[1], 0.5 * red[2], red[3], red[4], red[5]};
    grid_sum_finish<6>(v, partials, counter, thermo, false);
  }
}

// LAW 0: Lennard-Jones (velocities updated in place: no neighbour reads them);
// LAW 1: Spring-Dashpot (the dashpot reads v_j, so the kicked velocities go to
// a second buffer, like the drifted positions).
// thermo steps (ENERGY) carry 3 more accumulators: 2 blocks per SM, no spills
template <int LAW, bool ENERGY>
// thermo steps (ENERGY) too at 4 blocks/SM: with thermo every step (run()'s
// default) 0.439 ms vs 0.494 at 2 blocks (116 registers) despite a 56-byte spill
#ifndef TMD_ENERGY_MIN_BLOCKS
#define TMD_ENERGY_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kStepBlock, ENERGY ? TMD_ENERGY_MIN_BLOCKS : (LAW == 0 ? kStepMinBlocksLJ : kStepMinBlocksSD)) k_step(
    const double* __restrict__ pos, double* __restrict__ pos_out, const double* vel, double* vel_out, int64_t ld,
    int32_t n, const int32_t* __restrict__ nbr, int64_t ld_nbr, const int32_t* __restrict__ nnbr, LJFast lj,
    SDFast sd, Prune pr, Exports ex, double c, double dt, int phases, bool store_f, double* __restrict__ frc,
    int64_t ld_f, const double* __restrict__ xref, int64_t ld_ref, double* dispmax2, double* partials,
    unsigned int* counter, double* thermo, int64_t* st, double guard_lim2, bool skip_forces) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double red[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  double d2 = 0.0;
  // the row's first two quads: issued before anything else this atom needs
  int4 pre[2];
  if (i < n && !skip_forces) {
    const int4* __restrict__ row = reinterpret_cast<const int4*>(nbr) + i;
    pre[0] = ld_quad(row);
    pre[1] = pr.cap4 >= 8 ? ld_quad(row + ld_nbr) : make_int4(i, i, i, i);
  }
  // every per-atom load of the prologue is issued here, before the fail-fast
  // test below (whose loads would otherwise serialise in front of them)
  double xi = 0.0, yi = 0.0, zi = 0.0, xr = 0.0, yr = 0.0, zr = 0.0;
  int32_t seg_nn = 0, seg_nb = 0;
  if (i < n) {
    xi = pos[i];
    yi = pos[ld + i];
    zi = pos[2 * ld + i];
    if (xref) {
      xr = __ldcs(xref + i);
      yr = __ldcs(xref + ld_ref + i);
      zr = __ldcs(xref + 2 * ld_ref + i);
    }
    if (!skip_forces) {
      seg_nb = __ldcs(nnbr + i);
      seg_nn = pr.nnear ? __ldcs(pr.nnear + i) : seg_nb;
    }
    // the epilogue's velocities: into L2 now, so their DRAM latency is not
    // exposed after the force loop
    asm volatile("prefetch.global.L2 [%0];" ::"l"(vel + i));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(vel + ld + i));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(vel + 2 * ld + i));
  }
  // Fail fast: after an error of an earlier step (status word set) or when the
  // current positions violate the displacement guard (driver.py:115-125: the
  // reference raises before computing the step's forces), no atom is advanced:
  // the state stays the one the reference would raise on, and the host raises
  // at its next check.  Every block still takes part in the grid reduction.
  const bool guard_hit = !skip_forces && guard_lim2 > 0.0 && pr.disp2 && *pr.disp2 >= guard_lim2;
  // (a plain load: earlier launches' errors are visible at kernel start; an
  // error raised by another block of this launch may or may not be seen)
  const bool frozen = guard_hit || *st != TMD_OK;
  if (guard_hit && blockIdx.x == 0 && threadIdx.x == 0) raise_status(st, TMD_GUARD, 0);
  if (i < n && !frozen) {
    const double di2 = xref ? norm2_seq(sub_rn(xi, xr), sub_rn(yi, yr), sub_rn(zi, zr)) : 0.0;
    double fx, fy, fz, e = 0.0, w = 0.0;
    if (skip_forces) {  // F of this step was stored by the previous launch
      fx = frc[i];
      fy = frc[ld_f + i];
      fz = frc[2 * ld_f + i];
    } else {
      const RowSegs sg = row_segments(seg_nn, seg_nb, pr, di2);
      if (LAW == 0)
        lj_fast_atom<ENERGY>(pos, ld, i, xi, yi, zi, nbr, ld_nbr, sg, pr.cap4, lj, fx, fy, fz, e, w, st, pre);
      else
        sd_fast_atom<ENERGY>(pos, vel, ld, i, xi, yi, zi, nbr, ld_nbr, sg, pr.cap4, sd, fx, fy, fz, e, w, st, pre);
    }
    step_atom_tail<ENERGY>(i, xi, yi, zi, fx, fy, fz, e, w, pos_out, vel, vel_out, ld, ex, c, dt, phases,
                           store_f && !skip_forces, frc, ld_f, xref != nullptr, xr, yr, zr, red, d2);
  } else if (i < n) {
    // frozen: carry the state unchanged into the buffers the host swaps in
    if (phases & TMD_PHASE_NEXT) {
#pragma unroll
      for (int q = 0; q < 3; ++q) pos_out[q * ld + i] = pos[q * ld + i];
    }
    if (vel_out != vel) {
#pragma unroll
      for (int q = 0; q < 3; ++q) vel_out[q * ld + i] = vel[q * ld + i];
    }
  }
  step_block_finish<ENERGY>(phases, xref, d2, dispmax2, red, partials, counter, thermo);
}

// ---------------------------------------------------------------------------
// Spring-Dashpot over full lists, reference order (potential.py:80-93)
// ---------------------------------------------------------------------------
template <bool ENERGY>
__global__ void __launch_bounds__(128) k_force_sd(
    const double* __restrict__ pos, const double* __restrict__ vel, int64_t ld, int32_t n,
    const int32_t* __restrict__ nbr, int64_t ld_nbr, const int32_t* __restrict__ nnbr,
    int32_t cap, SDExact law, double* __restrict__ frc, int64_t ld_f, double* partials,
    unsigned int* counter, double* thermo, int64_t* st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double red[2] = {0.0, 0.0};
  if (i < n) {
    const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
    const double vix = vel[i], viy = vel[ld + i], viz = vel[2 * ld + i];
    const double rc2 = mul_rn(law.diam, law.diam);
    const int32_t cnt = nnbr[i];
    double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0, w = 0.0;
    for (int32_t k = 0; k < cnt; ++k) {
      const int32_t j = nbr[slot_index(k, i, ld_nbr)];
      const double dx = sub_rn(xi, pos[j]);
      const double dy = sub_rn(yi, pos[ld + j]);
      const double dz = sub_rn(zi, pos[2 * ld + j]);
      const double rsq = rsq_ref(dx, dy, dz);
      double px = 0.0, py = 0.0, pz = 0.0;
      if (rsq < rc2) {
        if (rsq == 0.0) report_singular(st, i, k);
        law.force(dx, dy, dz, rsq, vix, viy, viz, vel[j], vel[ld + j], vel[2 * ld + j], px, py, pz);
        if (ENERGY) {
          e += law.energy(rsq);
          w += px * dx + py * dy + pz * dz;
        }
      }
      if (k == 0) {
        fx = px; fy = py; fz = pz;
      } else {
        fx = add_rn(fx, px); fy = add_rn(fy, py); fz = add_rn(fz, pz);
      }
    }
    if (cnt < cap) {
      fx = add_rn(fx, 0.0); fy = add_rn(fy, 0.0); fz = add_rn(fz, 0.0);
    }
    frc[i] = fx;
    frc[ld_f + i] = fy;
    frc[2 * ld_f + i] = fz;
    red[0] = e;
    red[1] = w;
  }
  if (ENERGY) {
    __shared__ double sm[64];
    block_sum<2>(red, sm);
    double v[2] = {0.5 * red[0], 0.5 * red[1]};
    grid_sum_finish<2>(v, partials, counter, thermo, false);
  }
}

// ---------------------------------------------------------------------------
// half lists with reaction scatter (potential.py:187-191, 205-209)
// ---------------------------------------------------------------------------
template <int LAW, bool ENERGY>
__global__ void __launch_bounds__(128) k_force_half(
    const double* __restrict__ pos, const double* __restrict__ vel, int64_t ld, int32_t n,
    const int32_t* __restrict__ nbr, int64_t ld_nbr, const int32_t* __restrict__ nnbr,
    LJExact lj, SDExact sd, double rc2, double* __restrict__ frc, int64_t ld_f, double* partials,
    unsigned int* counter, double* thermo, int64_t* st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double red[2] = {0.0, 0.0};
  if (i < n) {
    const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
    double vix = 0, viy = 0, viz = 0;
    if (LAW == 1) { vix = vel[i]; viy = vel[ld + i]; viz = vel[2 * ld + i]; }
    const int32_t cnt = nnbr[i];
    double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0, w = 0.0;
    for (int32_t k = 0; k < cnt; ++k) {
      const int32_t j = nbr[slot_index(k, i, ld_nbr)];
      const double dx = sub_rn(xi, pos[j]);
      const double dy = sub_rn(yi, pos[ld + j]);
      const double dz = sub_rn(zi, pos[2 * ld + j]);
      const double rsq = rsq_ref(dx, dy, dz);
      if (!(rsq < rc2)) continue;
      if (rsq == 0.0) report_singular(st, i, k);
      double px, py, pz;
      if (LAW == 0) {
        double f = lj.scalar(rsq);
        px = mul_rn(f, dx); py = mul_rn(f, dy); pz = mul_rn(f, dz);
        if (ENERGY) e += lj.energy(rsq);
      } else {
        sd.force(dx, dy, dz, rsq, vix, viy, viz, vel[j], vel[ld + j], vel[2 * ld + j], px, py, pz);
        if (ENERGY) e += sd.energy(rsq);
      }
      if (ENERGY) w += px * dx + py * dy + pz * dz;
      fx = add_rn(fx, px); fy = add_rn(fy, py); fz = add_rn(fz, pz);
      if (j < n) {
        atomicAdd(frc + j, -px);
        atomicAdd(frc + ld_f + j, -py);
        atomicAdd(frc + 2 * ld_f + j, -pz);
      }
    }
    atomicAdd(frc + i, fx);
    atomicAdd(frc + ld_f + i, fy);
    atomicAdd(frc + 2 * ld_f + i, fz);
    red[0] = e;
    red[1] = w;
  }
  if (ENERGY) {
    __shared__ double sm[64];
    block_sum<2>(red, sm);
    double v[2] = {red[0], red[1]};
    grid_sum_finish<2>(v, partials, counter, thermo, false);
  }
}

// ---------------------------------------------------------------------------
// pair laws on arrays (API: law.pair_force / pair_energy)
// ---------------------------------------------------------------------------
__global__ void k_pair_force(int law, const double* __restrict__ d, const double* __restrict__ rsq,
                             const double* __restrict__ vi, const double* __restrict__ vj, int32_t n,
                             double p0, double p1, double p2, double* __restrict__ out) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double dx = d[3 * t], dy = d[3 * t + 1], dz = d[3 * t + 2];
  double fx, fy, fz;
  if (law == 0) {
    LJExact lj{p0, p1};
    double f = lj.scalar(rsq[t]);
    fx = mul_rn(f, dx); fy = mul_rn(f, dy); fz = mul_rn(f, dz);
  } else {
    SDExact sd{p0, p1, p2};
    double a0 = 0, a1 = 0, a2 = 0, b0 = 0, b1 = 0, b2 = 0;
    if (vi && vj) {
      a0 = vi[3 * t]; a1 = vi[3 * t + 1]; a2 = vi[3 * t + 2];
      b0 = vj[3 * t]; b1 = vj[3 * t + 1]; b2 = vj[3 * t + 2];
    }
    sd.force(dx, dy, dz, rsq[t], a0, a1, a2, b0, b1, b2, fx, fy, fz);
  }
  out[3 * t] = fx;
  out[3 * t + 1] = fy;
  out[3 * t + 2] = fz;
}

__global__ void k_pair_energy(int law, const double* __restrict__ rsq, int32_t n, double p0, double p1,
                              double p2, double* __restrict__ out) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (law == 0) {
    out[t] = LJExact{p0, p1}.energy(rsq[t]);
  } else {
    out[t] = SDExact{p0, p1, p2}.energy(rsq[t]);
  }
}

}  // namespace tmd

using namespace tmd;

namespace {
constexpr int kB = 128;
}

extern "C" int tmd_force_lj(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_nbr,
                            int64_t ld_nbr, const int32_t* d_nnbr, int32_t cap, double rc2,
                            double eps, double sigma6, uint32_t flags, double* d_frc, int64_t ld_f,
                            double* d_thermo, int64_t* d_status, void* stream) {
  cudaStream_t s = as_stream(stream);
  const bool energy = flags & TMD_F_ENERGY;
  if (n_local <= 0) {
    if (energy) TMD_CUDA_TRY(cudaMemsetAsync(d_thermo, 0, 2 * sizeof(double), s), "force_lj");
    return TMD_OK;
  }
  const int g = grid_for(n_local, kB);
  ReduceScratch rs{};
  if (energy && reduce_scratch(&rs, g, 2, s) != TMD_OK) return TMD_ERR_CUDA;
  if (flags & TMD_F_EXACT) {
    LJExact law{eps, sigma6};
    if (energy)
      k_force_lj_exact<true><<<g, kB, 0, s>>>(d_pos, ld, n_local, d_nbr, ld_nbr, d_nnbr, cap, rc2,
                                              law, d_frc, ld_f, rs.partials, rs.counter, d_thermo,
                                              d_status);
    else
      k_force_lj_exact<false><<<g, kB, 0, s>>>(d_pos, ld, n_local, d_nbr, ld_nbr, d_nnbr, cap, rc2,
                                               law, d_frc, ld_f, nullptr, nullptr, nullptr,
                                               d_status);
  } else {
    const LJFast p = lj_fast_params(rc2, eps, sigma6);
    const int gf = grid_for(n_local, kLJBlock);
    ReduceScratch rf{};
    if (energy && reduce_scratch(&rf, gf, 2, s) != TMD_OK) return TMD_ERR_CUDA;
    if (energy)
      k_force_lj_fast<true><<<gf, kLJBlock, 0, s>>>(d_pos, ld, n_local, d_nbr, ld_nbr, d_nnbr, p, d_frc, ld_f,
                                                    rf.partials, rf.counter, d_thermo, d_status);
    else
      k_force_lj_fast<false><<<gf, kLJBlock, 0, s>>>(d_pos, ld, n_local, d_nbr, ld_nbr, d_nnbr, p, d_frc, ld_f,
                                                     nullptr, nullptr, nullptr, d_status);
  }
  TMD_LAUNCH_CHECK("force_lj");
  return TMD_OK;
}

// Shared body of the fused step entries (argument checks, exports, pruning).
static int launch_step(int law, const double* d_pos, double* d_pos_out, const double* d_vel, double* d_vel_out,
                       int64_t ld, int32_t n_local, const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr,
                       const int32_t* d_nnear, int32_t cap, double near_margin, const double* d_prune_disp2,
                       const int32_t* d_ex_start, const int32_t* d_ex_rank, const int32_t* d_ex_slot,
                       const double* d_ex_sh, int64_t n_ex, int32_t n_peers, double* const* h_peer_base,
                       const int64_t* h_peer_ld, const double* h_ex_border, const LJFast& lj, const SDFast& sd,
                       double half_dt_over_m, double dt, int32_t phases, uint32_t flags, double* d_frc, int64_t ld_f,
                       const double* d_xref, int64_t ld_ref, double* d_dispmax2, double* d_thermo,
                       int64_t* d_status, double guard_lim2, cudaStream_t s) {
  const bool skip = flags & TMD_F_SKIP_FORCES;
  const bool energy = (flags & TMD_F_ENERGY) && !skip;
  const bool store_f = flags & TMD_F_STORE_FORCES;
  if (n_local <= 0) {
    if (energy) TMD_CUDA_TRY(cudaMemsetAsync(d_thermo, 0, 6 * sizeof(double), s), "step");
    return TMD_OK;
  }
  if ((d_nnear && (!d_prune_disp2 || !d_xref)) || ((store_f || skip) && !d_frc) ||
      ((phases & TMD_PHASE_NEXT) && !d_pos_out) || !d_vel || !d_vel_out || (skip && (phases & TMD_PHASE_FINAL)))
    return TMD_ERR_ARG;
  Exports ex;
  int rc = make_exports(d_ex_start, d_ex_rank, d_ex_slot, d_ex_sh, n_ex, n_peers, h_peer_base, h_peer_ld,
                        h_ex_border, d_xref, &ex);
  if (rc != TMD_OK) return rc;
  Prune pr{};
  pr.nnear = d_nnear;
  pr.disp2 = d_prune_disp2;
  pr.cap4 = (cap + 3) / 4 * 4;
  // TMD_F_NO_PRUNE (tests): scan both segments of every row
  pr.lim = (flags & TMD_F_NO_PRUNE) ? -1.0 : near_margin - 1e-9;
  const int g = grid_for(n_local, kStepBlock);
  ReduceScratch rs{};
  if (energy && reduce_scratch(&rs, g, 6, s) != TMD_OK) return TMD_ERR_CUDA;
#define TMD_STEP(L, E)                                                                                          \
  k_step<L, E><<<g, kStepBlock, 0, s>>>(d_pos, d_pos_out, d_vel, d_vel_out, ld, n_local, d_nbr, ld_nbr, d_nnbr, lj, \
                                      sd, pr, ex, half_dt_over_m, dt, phases, store_f, d_frc, ld_f, d_xref,      \
                                      ld_ref, d_dispmax2, E ? rs.partials : nullptr, E ? rs.counter : nullptr,  \
                                      E ? d_thermo : nullptr, d_status, guard_lim2, skip)
  if (law == 0) {
    if (energy) TMD_STEP(0, true); else TMD_STEP(0, false);
  } else {
    if (energy) TMD_STEP(1, true); else TMD_STEP(1, false);
  }
#undef TMD_STEP
  TMD_LAUNCH_CHECK(law == 0 ? "step_lj" : "step_sd");
  return TMD_OK;
}

extern "C" int tmd_step_lj(const double* d_pos, double* d_pos_out, double* d_vel, int64_t ld,
                           int32_t n_local, const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr,
                           const int32_t* d_nnear, int32_t cap, double near_margin,
                           const double* d_prune_disp2, const int32_t* d_ex_start, const int32_t* d_ex_rank,
                           const int32_t* d_ex_slot, const double* d_ex_sh, int64_t n_ex, int32_t n_peers,
                           double* const* h_peer_base, const int64_t* h_peer_ld, const double* h_ex_border,
                           double rc2, double eps, double sigma6,
                           double half_dt_over_m, double dt, int32_t phases, uint32_t flags,
                           double* d_frc, int64_t ld_f, const double* d_xref, int64_t ld_ref,
                           double* d_dispmax2, double* d_thermo, int64_t* d_status, double guard_lim2,
                           void* stream) {
  return launch_step(0, d_pos, d_pos_out, d_vel, d_vel, ld, n_local, d_nbr, ld_nbr, d_nnbr, d_nnear, cap, near_margin,
                     d_prune_disp2, d_ex_start, d_ex_rank, d_ex_slot, d_ex_sh, n_ex, n_peers, h_peer_base, h_peer_ld,
                     h_ex_border, lj_fast_params(rc2, eps, sigma6), SDFast{}, half_dt_over_m, dt, phases, flags,
                     d_frc, ld_f, d_xref, ld_ref, d_dispmax2, d_thermo, d_status, guard_lim2, as_stream(stream));
}

extern "C" int tmd_step_sd(const double* d_pos, double* d_pos_out, const double* d_vel, double* d_vel_out, int64_t ld,
                           int32_t n_local, const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr,
                           const int32_t* d_nnear, int32_t cap, double near_margin,
                           const double* d_prune_disp2, const int32_t* d_ex_start, const int32_t* d_ex_rank,
                           const int32_t* d_ex_slot, const double* d_ex_sh, int64_t n_ex, int32_t n_peers,
                           double* const* h_peer_base, const int64_t* h_peer_ld, const double* h_ex_border,
                           double stiffness, double damping, double diameter,
                           double half_dt_over_m, double dt, int32_t phases, uint32_t flags,
                           double* d_frc, int64_t ld_f, const double* d_xref, int64_t ld_ref,
                           double* d_dispmax2, double* d_thermo, int64_t* d_status, double guard_lim2,
                           void* stream) {
  if (d_vel == d_vel_out && (phases & (TMD_PHASE_FINAL | TMD_PHASE_NEXT))) return TMD_ERR_ARG;
  const SDFast sd{diameter * diameter, diameter, stiffness, damping, 0.5 * stiffness};
  return launch_step(1, d_pos, d_pos_out, d_vel, d_vel_out, ld, n_local, d_nbr, ld_nbr, d_nnbr, d_nnear, cap,
                     near_margin, d_prune_disp2, d_ex_start, d_ex_rank, d_ex_slot, d_ex_sh, n_ex, n_peers, h_peer_base,
                     h_peer_ld, h_ex_border, LJFast{}, sd, half_dt_over_m, dt, phases, flags, d_frc, ld_f, d_xref,
                     ld_ref, d_dispmax2, d_thermo, d_status, guard_lim2, as_stream(stream));
}

extern "C" int tmd_force_sd(const double* d_pos, const double* d_vel, int64_t ld, int32_t n_local,
                            const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr, int32_t cap,
                            double stiffness, double damping, double diameter, uint32_t flags,
                            double* d_frc, int64_t ld_f, double* d_thermo, int64_t* d_status,
                            void* stream) {
  cudaStream_t s = as_stream(stream);
  const bool energy = flags & TMD_F_ENERGY;
  if (n_local <= 0) {
    if (energy) TMD_CUDA_TRY(cudaMemsetAsync(d_thermo, 0, 2 * sizeof(double), s), "force_sd");
    return TMD_OK;
  }
  const int g = grid_for(n_local, kB);
  ReduceScratch rs{};
  if (energy && reduce_scratch(&rs, g, 2, s) != TMD_OK) return TMD_ERR_CUDA;
  SDExact law{stiffness, damping, diameter};
  if (energy)
    k_force_sd<true><<<g, kB, 0, s>>>(d_pos, d_vel, ld, n_local, d_nbr, ld_nbr, d_nnbr, cap, law,
                                      d_frc, ld_f, rs.partials, rs.counter, d_thermo, d_status);
  else
    k_force_sd<false><<<g, kB, 0, s>>>(d_pos, d_vel, ld, n_local, d_nbr, ld_nbr, d_nnbr, cap, law,
                                       d_frc, ld_f, nullptr, nullptr, nullptr, d_status);
  TMD_LAUNCH_CHECK("force_sd");
  return TMD_OK;
}

extern "C" int tmd_force_half(const double* d_pos, const double* d_vel, int64_t ld, int32_t n_local,
                              const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr,
                              int32_t law, double p0, double p1, double p2, uint32_t flags,
                              double* d_frc, int64_t ld_f, double* d_thermo, int64_t* d_status,
                              void* stream) {
  cudaStream_t s = as_stream(stream);
  const bool energy = flags & TMD_F_ENERGY;
  for (int c = 0; c < 3; ++c)
    TMD_CUDA_TRY(cudaMemsetAsync(d_frc + c * ld_f, 0, sizeof(double) * (size_t)(n_local > 0 ? n_local : 0), s),
                 "force_half");
  if (n_local <= 0) {
    if (energy) TMD_CUDA_TRY(cudaMemsetAsync(d_thermo, 0, 2 * sizeof(double), s), "force_half");
    return TMD_OK;
  }
  const int g = grid_for(n_local, kB);
  ReduceScratch rs{};
  if (energy && reduce_scratch(&rs, g, 2, s) != TMD_OK) return TMD_ERR_CUDA;
  // law 0: LJ (p0 eps, p1 sigma6, p2 cutoff); law 1: SD (p0 K, p1 gamma, p2 diameter)
  LJExact lj{p0, p1};
  SDExact sd{p0, p1, p2};
  double rc2 = p2 * p2;
  if (law == 0) {
    if (energy)
      k_force_half<0, true><<<g, kB, 0, s>>>(d_pos, d_vel, ld, n_local, d_nbr, ld_nbr, d_nnbr, lj, sd,
                                             rc2, d_frc, ld_f, rs.partials, rs.counter, d_thermo, d_status);
    else
      k_force_half<0, false><<<g, kB, 0, s>>>(d_pos, d_vel, ld, n_local, d_nbr, ld_nbr, d_nnbr, lj,
                                              sd, rc2, d_frc, ld_f, nullptr, nullptr, nullptr, d_status);
  } else {
    if (energy)
      k_force_half<1, true><<<g, kB, 0, s>>>(d_pos, d_vel, ld, n_local, d_nbr, ld_nbr, d_nnbr, lj, sd,
                                             rc2, d_frc, ld_f, rs.partials, rs.counter, d_thermo, d_status);
    else
      k_force_half<1, false><<<g, kB, 0, s>>>(d_pos, d_vel, ld, n_local, d_nbr, ld_nbr, d_nnbr, lj,
                                              sd, rc2, d_frc, ld_f, nullptr, nullptr, nullptr, d_status);
  }
  TMD_LAUNCH_CHECK("force_half");
  return TMD_OK;
}

extern "C" int tmd_pair_force(int32_t law, const double* d_delta, const double* d_rsq,
                              const double* d_vi, const double* d_vj, int32_t n, double p0, double p1,
                              double p2, double* d_out, void* stream) {
  if (n <= 0) return TMD_OK;
  k_pair_force<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(law, d_delta, d_rsq, d_vi, d_vj, n,
                                                                p0, p1, p2, d_out);
  TMD_LAUNCH_CHECK("pair_force");
  return TMD_OK;
}

extern "C" int tmd_pair_energy(int32_t law, const double* d_rsq, int32_t n, double p0, double p1,
                               double p2, double* d_out, void* stream) {
  if (n <= 0) return TMD_OK;
  k_pair_energy<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(law, d_rsq, n, p0, p1, p2, d_out);
  TMD_LAUNCH_CHECK("pair_energy");
  return TMD_OK;
}

// ---------------------------------------------------------------------------
// Batched step loop (the production run between two epochs): the launches of
// steps k0 .. k1-1 issued from here, one host call per batch instead of one
// Python call per step.  Each step's arguments follow from the step index
// exactly as driver.Simulation derives them (buffer parity, thermo row, guard
// slot, flags, whether the next step refreshes ghosts, the P > 1 barrier).
// ---------------------------------------------------------------------------
#include <map>
#include <mutex>
#include <vector>

namespace {
struct LaunchTimes {
  std::vector<cudaEvent_t> ev;  // 2 per launch of the last timed batch
  int used = 0;
};
std::mutex g_times_mu;
std::map<cudaStream_t, LaunchTimes> g_times;
}  // namespace

extern "C" int tmd_run_steps(const TmdStepRun* r, int32_t k0, int32_t k1, void* stream) {
  if (!r || k1 < k0 || (r->law != 0 && r->law != 1) || !r->pos_a || !r->pos_b || !r->vel_a ||
      (r->law == 1 && !r->vel_b) || r->thermo_every < 1 || r->reneigh < 1 || !r->dispmax2 || !r->thermo)
    return TMD_ERR_ARG;
  if (k1 == k0) return TMD_OK;
  cudaStream_t s = as_stream(stream);
  const LJFast lj = r->law == 0 ? lj_fast_params(r->p0, r->p1, r->p2) : LJFast{};
  const SDFast sd = r->law == 1 ? SDFast{r->p2 * r->p2, r->p2, r->p0, r->p1, 0.5 * r->p0} : SDFast{};
  LaunchTimes* times = nullptr;
  if (r->time_launches) {
    // appended to the stream's list until tmd_run_launch_times reads it
    std::lock_guard<std::mutex> lock(g_times_mu);
    times = &g_times[s];
    const size_t need = times->used + 2 * (size_t)(k1 - k0);
    while (times->ev.size() < need) {
      cudaEvent_t e;
      TMD_CUDA_TRY(cudaEventCreate(&e), "run_steps events");
      times->ev.push_back(e);
    }
  }
  const bool have_ex = r->ex_start != nullptr;
  for (int32_t k = k0; k < k1; ++k) {
    const int odd = (k - k0) & 1;
    const int32_t phases = TMD_PHASE_FINAL | (k < r->k_last ? TMD_PHASE_NEXT : 0);
    uint32_t flags = 0;
    if (k % r->thermo_every == 0 || k == r->k_last) flags |= TMD_F_ENERGY;
    if (r->store_every || k == r->k_last) flags |= TMD_F_STORE_FORCES;
    const bool refresh = have_ex && k < r->k_last && (k + 1) % r->reneigh != 0;
    const int parity = (int)((k - r->epoch_step) & 1);
    const double* pos = odd ? r->pos_b : r->pos_a;
    double* pos_out = (phases & TMD_PHASE_NEXT) ? (odd ? r->pos_a : r->pos_b) : nullptr;
    const double* vel = r->law == 1 && odd ? r->vel_b : r->vel_a;
    double* vel_out = r->law == 1 ? (odd ? r->vel_a : r->vel_b) : r->vel_a;
    const double guard = (k == k0 && r->rebuild_at_k0) ? 0.0 : r->guard_lim2;
    double* disp = r->dispmax2 + ((phases & TMD_PHASE_NEXT) ? k + 1 : 0);
    if (times) TMD_CUDA_TRY(cudaEventRecord(times->ev[times->used++], s), "run_steps event");
    const uint64_t* base = parity ? r->peer_base1 : r->peer_base0;
    const int rc = launch_step(
        (int)r->law, pos, pos_out, vel, vel_out, r->ld, (int32_t)r->n_local, r->nbr, r->ld_nbr, r->nnbr, r->nnear,
        (int32_t)r->cap, r->near_margin, r->dispmax2 + k, refresh ? r->ex_start : nullptr,
        refresh ? r->ex_rank : nullptr, refresh ? r->ex_slot : nullptr, refresh ? r->ex_sh : nullptr,
        refresh ? r->n_ex : 0, refresh ? (int32_t)r->n_peers : 0,
        refresh ? reinterpret_cast<double* const*>(base) : nullptr, refresh ? r->peer_ld : nullptr,
        refresh ? r->ex_border : nullptr, lj, sd, r->half_dt_over_m, r->dt, phases, flags, r->frc, r->ld_f, r->xref,
        r->ld_ref, disp, r->thermo + (int64_t)k * r->thermo_stride, r->status, guard, s);
    if (rc != TMD_OK) return rc;
    if (times) TMD_CUDA_TRY(cudaEventRecord(times->ev[times->used++], s), "run_steps event");
    if (r->size > 1 && have_ex && k < r->k_last) {
      const int rc2 = tmd_peer_sync(r->barrier_epoch0 + (k - k0) + 1, (int32_t)r->rank, (int32_t)r->size,
                                    reinterpret_cast<int64_t* const*>(r->mailboxes), r->dispmax2 + k + 1,
                                    r->barrier_timeout_s, r->status, stream);
      if (rc2 != TMD_OK) return rc2;
    }
  }
  return TMD_OK;
}

extern "C" int tmd_run_launch_times(void* stream, float* h_ms, int32_t n) {
  std::lock_guard<std::mutex> lock(g_times_mu);
  auto it = g_times.find(as_stream(stream));
  if (it == g_times.end()) return 0;
  const int m = it->second.used / 2 < n ? it->second.used / 2 : n;
  for (int q = 0; q < m; ++q)
    if (h_ms && cudaEventElapsedTime(h_ms + q, it->second.ev[2 * q], it->second.ev[2 * q + 1]) != cudaSuccess)
      return -1;
  it->second.used = 0;
  return m;
}
