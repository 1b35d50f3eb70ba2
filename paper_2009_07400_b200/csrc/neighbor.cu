// K2 — Verlet-list build over the 27-cell stencil (reference: _fill_lists /
// build_neighbor_lists, neighbor.py:92-194) and K6 — displacement since the
// last rebuild (max_displacement_since_rebuild, neighbor.py:197-206).
//
// List layout (both builders): "quad-interleaved neighbor-major".  Slot k of
// local i lives at nbr[((k >> 2) * ld_nbr + i) * 4 + (k & 3)]: the four slots
// 4q..4q+3 of an atom are one 16-byte int4, and the int4s of 32 consecutive
// atoms are one contiguous 512-byte run, so a warp fetches four candidates per
// atom with one fully coalesced vector load.  Unused slots of the last quad
// hold i itself (a valid address, masked by the count).
//
// The 27-cell stencil is walked as 9 contiguous runs of the cell table: for a
// fixed (dx, dy), the cells dz = -1, 0, +1 have consecutive ids, so their atoms
// are one range of cell_atoms (ascending inside each cell) — exactly the
// reference's candidate order (neighbor.py:30-33, 81-86, 127-131).
//
//  * reference order (tmd_build_lists): rows identical slot for slot to the
//    reference; the rsq predicate is evaluated in the reference's operation
//    order, so membership is bit-exact.
//  * tiered order (tmd_build_lists_tiered, production): same membership,
//    rows bucketed by distance tier R_t = rc + m_t (m_t <= skin) and the
//    cumulative count per tier stored in tcnt[t * ld_nbr + i].  A force pass
//    whose atoms moved at most d since the build only needs the prefix of
//    tier t with m_t >= 2 d: every pair beyond it is farther than rc.
#include "tmd_common.cuh"

namespace tmd {

struct Stencil {
  int g0, g1, g2;
};

struct Cells {
  const int32_t* cell_of;
  const int32_t* cell_start;
  const int32_t* cell_atoms;
  const double* cp;  // positions in cell order
  int64_t ld_cp;
  Stencil g;
};

constexpr int kMaxTiers = 8;
constexpr int kTierShift = 28;  // staged entries are j | tier << 28 (n_total < 2^28)

struct Tiers {
  double r2[kMaxTiers];  // ascending squared tier radii, padded with the list radius^2
  int nt;
};

// Warp-cooperative list build.  A warp owns 32 consecutive locals (with the
// production cell-ordered store: one or two cells) and builds their rows one
// atom at a time: the 32 lanes sweep the atom's 27-cell stencil, flattened
// into one sequence of candidates (9 contiguous z-runs of the cell table), 32
// consecutive candidates per step — coalesced position loads, every lane busy,
// no divergent loop bounds; the loads of step s+1 are issued before step s is
// reduced.  Accepted candidates keep the reference's order (ballot + popc
// prefix); tiered rows are then bucketed by distance tier with
// __match_any_sync ranks.  The finished row is written by the warp as whole
// int4 quads (the two quads sharing a 32-byte sector belong to consecutive
// atoms of the same warp, written microseconds apart, so L2 merges them).
struct Cand {
  int32_t j;
  double x, y, z;
};

// Candidate c of the flattened stencil: its run r is the last with run_p[r] <= c
// (run_p ascending; empty runs share the next run's prefix), found by a
// binary search in the warp's shared run table.
__device__ __forceinline__ Cand load_cand(const Cells& C, const int32_t* __restrict__ run_s,
                                          const int32_t* __restrict__ run_p, int nruns, int32_t c, int32_t total) {
  Cand r{-1, 0.0, 0.0, 0.0};
  if (c < total) {
    int lo = 0, hi = nruns - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (run_p[mid] <= c) lo = mid;
      else hi = mid - 1;
    }
    const int32_t k = run_s[lo] + (c - run_p[lo]);
    r.j = __ldg(C.cell_atoms + k);
    r.x = __ldg(C.cp + k);
    r.y = __ldg(C.cp + C.ld_cp + k);
    r.z = __ldg(C.cp + 2 * C.ld_cp + k);
  }
  return r;
}

constexpr int kRunTable = 64;  // per-warp shared run table: starts [0, 32), prefixes [32, 64)

template <bool TIERED>
__global__ void __launch_bounds__(128) k_build_warp(
    const double* __restrict__ pos, int64_t ld, int32_t n_local, Cells C, int H, double rsq_max, int half,
    Tiers T, int32_t cap, int32_t cap_s, int32_t* __restrict__ nbr, int64_t ld_nbr, int32_t* __restrict__ tcnt,
    int32_t* __restrict__ nnbr, int64_t* __restrict__ st) {
  extern __shared__ int32_t smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  int32_t* row = smem + (size_t)w * (2 * cap_s + kRunTable);  // the current row, a scratch row, runs
  int32_t* tmp = row + cap_s;
  int32_t* run_s = tmp + cap_s;
  int32_t* run_p = run_s + 32;
  const int32_t a0 = (blockIdx.x * wpb + w) * 32;
  if (a0 >= n_local) return;
  const unsigned lt = (1u << lane) - 1u;
  long long r2b[kMaxTiers];  // tier radii^2 as ordered bit patterns
#pragma unroll
  for (int q = 0; q < kMaxTiers; ++q) r2b[q] = __double_as_longlong(T.r2[q]);
  const Stencil g = C.g;
  const int side = 2 * H + 1, nruns = side * side;  // (2H+1)^2 z-runs of 2H+1 cells
  int4* out4 = reinterpret_cast<int4*>(nbr);
  int last_cell = -1;
  int32_t total = 0;
  for (int a = 0; a < 32; ++a) {
    const int32_t i = a0 + a;
    if (i >= n_local) break;
    const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
    const int cid = C.cell_of[i];
    if (cid != last_cell) {  // atoms of one cell share the stencil: rebuild the run table on a change
      last_cell = cid;
      const int c2 = cid % g.g2, c1 = (cid / g.g2) % g.g1, c0 = cid / (g.g1 * g.g2);
      const int zlo = c2 - H > 0 ? c2 - H : 0, zhi = c2 + H < g.g2 ? c2 + H : g.g2 - 1;
      // lane r < nruns: z-run r in stencil order (dx slowest, then dy)
      int32_t rs = 0, rl = 0;
      if (lane < nruns) {
        const int ca = c0 - H + lane / side, cb = c1 - H + lane % side;
        if (ca >= 0 && ca < g.g0 && cb >= 0 && cb < g.g1) {
          const int base = (ca * g.g1 + cb) * g.g2;
          rs = __ldg(C.cell_start + base + zlo);
          rl = __ldg(C.cell_start + base + zhi + 1) - rs;
        }
      }
      int32_t incl = rl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      __syncwarp();
      run_s[lane] = rs;
      run_p[lane] = incl - rl;
      total = __shfl_sync(0xffffffffu, incl, nruns - 1);
      __syncwarp();
    }
    int32_t cnt = 0;
    // per-lane tier histogram, 16-bit fields packed in two 64-bit words
    // (tiers 0-3, 4-7); reduced across the warp once per atom
    unsigned long long h0 = 0ull, h1 = 0ull;
    int32_t* out = TIERED ? tmp : row;
    Cand nx = load_cand(C, run_s, run_p, nruns, lane, total);
    for (int32_t base = 0; base < total; base += 32) {
      const Cand cur = nx;
      nx = load_cand(C, run_s, run_p, nruns, base + 32 + lane, total);  // next step in flight
      bool acc = false;
      double rsq = 0.0;
      if (cur.j >= 0) {
        rsq = rsq_ref(sub_rn(xi, cur.x), sub_rn(yi, cur.y), sub_rn(zi, cur.z));
        acc = (half ? (cur.j >= n_local || cur.j > i) : (cur.j != i)) && rsq < rsq_max;
      }
      const unsigned m = __ballot_sync(0xffffffffu, acc);
      const int32_t p = cnt + __popc(m & lt);
      if (acc) {
        int t = 0;
        if (TIERED) {
          // non-negative doubles order like their bit patterns: integer compares
          const long long b = __double_as_longlong(rsq);
#pragma unroll
          for (int q = 0; q < kMaxTiers - 1; ++q) t += (b < r2b[q]) ? 0 : 1;
          if (t < 4) h0 += 1ull << (16 * t);
          else h1 += 1ull << (16 * (t - 4));
        }
        if (p < cap) out[p] = TIERED ? (cur.j | (t << kTierShift)) : cur.j;
      }
      cnt += __popc(m);
    }
    int32_t tc[kMaxTiers];
    if (TIERED) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        h0 += __shfl_xor_sync(0xffffffffu, h0, o);
        h1 += __shfl_xor_sync(0xffffffffu, h1, o);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        tc[q] = (int32_t)((h0 >> (16 * q)) & 0xffffull);
        tc[q + 4] = (int32_t)((h1 >> (16 * q)) & 0xffffull);
      }
    }
    if (lane == 0) nnbr[i] = cnt;
    if (cnt > cap) {
      if (lane == 0) need_capacity(st, cnt);
      continue;
    }
    __syncwarp();
    if (TIERED) {
      int32_t off[kMaxTiers];
      int32_t run = 0;
#pragma unroll
      for (int q = 0; q < kMaxTiers; ++q) {
        off[q] = run;
        run += tc[q];
        if (lane == q && q < T.nt) tcnt[(int64_t)q * ld_nbr + i] = run;
      }
      for (int32_t e0 = 0; e0 < cnt; e0 += 32) {
        const int32_t e = e0 + lane;
        const bool v = e < cnt;
        const int32_t val = v ? tmp[e] : 0;
        const int t = v ? (val >> kTierShift) : kMaxTiers;
        const unsigned peers = __match_any_sync(0xffffffffu, t);
        int32_t dst = __popc(peers & lt);
#pragma unroll
        for (int q = 0; q < kMaxTiers; ++q) dst += (t == q) ? off[q] : 0;
        if (v) row[dst] = val & ((1 << kTierShift) - 1);
#pragma unroll
        for (int q = 0; q < kMaxTiers; ++q) off[q] += __popc(__ballot_sync(0xffffffffu, v && t == q));
      }
      __syncwarp();
    }
    // the row as whole quads, lane q storing quad q (padding slots hold i)
    for (int32_t q = lane; 4 * q < cnt; q += 32) {
      const int32_t k = 4 * q;
      out4[(int64_t)q * ld_nbr + i] = make_int4(row[k], k + 1 < cnt ? row[k + 1] : i,
                                                k + 2 < cnt ? row[k + 2] : i, k + 3 < cnt ? row[k + 3] : i);
    }
    __syncwarp();
  }
}

__global__ void k_max_disp2(const double* __restrict__ pos, int64_t ld, const double* __restrict__ ref,
                            int64_t ld_ref, int32_t n, double* __restrict__ out) {
  double m = 0.0;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double dx = sub_rn(pos[i], ref[i]);
    double dy = sub_rn(pos[ld + i], ref[ld_ref + i]);
    double dz = sub_rn(pos[2 * ld + i], ref[2 * ld_ref + i]);
    m = fmax(m, norm2_seq(dx, dy, dz));
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

}  // namespace tmd

using namespace tmd;

static Cells make_cells(const int32_t* cell_of, const int32_t* cell_start, const int32_t* cell_atoms,
                        const double* cell_pos, int64_t ld_cp, const int32_t* h_dims, int shell) {
  Cells C;
  C.cell_of = cell_of;
  C.cell_start = cell_start;
  C.cell_atoms = cell_atoms;
  C.cp = cell_pos;
  C.ld_cp = ld_cp;
  C.g = Stencil{h_dims[0] + 2 * shell, h_dims[1] + 2 * shell, h_dims[2] + 2 * shell};
  return C;
}

static bool make_tiers(const double* h_tier_r2, int32_t n_tiers, Tiers* T) {
  if (!h_tier_r2 || n_tiers < 1 || n_tiers > kMaxTiers) return false;
  for (int q = 0; q < kMaxTiers; ++q) T->r2[q] = h_tier_r2[q < n_tiers ? q : n_tiers - 1];
  T->nt = n_tiers;
  return true;
}

template <bool TIERED>
static int launch_build(const double* d_pos, int64_t ld, int32_t n_local, const Cells& C, int H, double rsq_max,
                        int32_t half, const Tiers& T, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                        int32_t* d_tcnt, int32_t* d_nnbr, int64_t* d_status, cudaStream_t s) {
  // shared memory: the current row and a scratch row per warp
  const int32_t cap_s = cap < 1 ? 1 : cap;
  int wpb = 4;
  while (wpb > 1 && (size_t)wpb * (2 * cap_s + kRunTable) * 4 > 200 * 1024) wpb >>= 1;
  const size_t smem = (size_t)wpb * (2 * cap_s + kRunTable) * 4;
  if (smem > 220 * 1024) return TMD_ERR_ARG;
  TMD_CUDA_TRY(cudaFuncSetAttribute(k_build_warp<TIERED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "build_lists smem");
  const int64_t warps = ((int64_t)n_local + 31) / 32;
  const int blocks = (int)((warps + wpb - 1) / wpb);
  k_build_warp<TIERED><<<blocks, 32 * wpb, smem, s>>>(d_pos, ld, n_local, C, H, rsq_max, half, T, cap, cap_s, d_nbr,
                                                      ld_nbr, d_tcnt, d_nnbr, d_status);
  TMD_LAUNCH_CHECK("build_lists");
  return TMD_OK;
}

extern "C" int tmd_build_lists(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_cell_of,
                               const int32_t* d_cell_start, const int32_t* d_cell_atoms,
                               const double* d_cell_pos, int64_t ld_cp, const int32_t* h_dims,
                               double rsq_max, int32_t half, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                               int32_t* d_nnbr, int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!h_dims || !d_cell_pos || cap < 0 || ld_nbr < n_local) return TMD_ERR_ARG;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims, 1);
  Tiers T{};
  T.nt = 1;
  return launch_build<false>(d_pos, ld, n_local, C, 1, rsq_max, half, T, cap, d_nbr, ld_nbr, nullptr, d_nnbr,
                             d_status, as_stream(stream));
}

extern "C" int tmd_build_lists_tiered(const double* d_pos, int64_t ld, int32_t n_local,
                                      const int32_t* d_cell_of, const int32_t* d_cell_start,
                                      const int32_t* d_cell_atoms, const double* d_cell_pos,
                                      int64_t ld_cp, const int32_t* h_dims, int32_t shell,
                                      const double* h_tier_r2, int32_t n_tiers, int32_t cap, int32_t* d_nbr,
                                      int64_t ld_nbr, int32_t* d_tcnt, int32_t* d_nnbr, int64_t* d_status,
                                      void* stream) {
  if (n_local <= 0) return TMD_OK;
  Tiers T;
  if (!h_dims || !d_cell_pos || !make_tiers(h_tier_r2, n_tiers, &T) || cap < 0 || ld_nbr < n_local ||
      ld_cp >= (1ll << kTierShift) || shell < 1 || (2 * shell + 1) * (2 * shell + 1) > 32)
    return TMD_ERR_ARG;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims, shell);
  return launch_build<true>(d_pos, ld, n_local, C, shell, T.r2[T.nt - 1], 0, T, cap, d_nbr, ld_nbr, d_tcnt, d_nnbr,
                            d_status, as_stream(stream));
}

extern "C" int tmd_max_disp2(const double* d_pos, int64_t ld, const double* d_xref, int64_t ld_ref,
                             int32_t n, double* d_dispmax2, void* stream) {
  if (n <= 0) return TMD_OK;
  const int B = 256;
  int g = grid_for(n, B);
  if (g > 4 * sm_count()) g = 4 * sm_count();
  k_max_disp2<<<g, B, 0, as_stream(stream)>>>(d_pos, ld, d_xref, ld_ref, n, d_dispmax2);
  TMD_LAUNCH_CHECK("max_disp2");
  return TMD_OK;
}
