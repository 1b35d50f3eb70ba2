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
#include <cstdlib>

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
  const int32_t* order;  // builder thread t -> local atom (null: t itself)
};

constexpr int kMaxTiers = 8;

struct Tiers {
  double r2[kMaxTiers];  // ascending squared tier radii, padded with the list radius^2
  int nt;
};

// Four accepted candidates are packed in registers and stored as one int4:
// every quad (and 32-byte sector) of a reference-order row is written once
// and completely.
struct QuadWriter {
  int4* out;  // quad q of atom i at out[q * ld + i]
  int64_t ld;
  int32_t i;
  int32_t a0, a1, a2, a3;
  __device__ __forceinline__ void put(int32_t o, int32_t j) {
    const int r = o & 3;
    a0 = r == 0 ? j : a0;
    a1 = r == 1 ? j : a1;
    a2 = r == 2 ? j : a2;
    a3 = r == 3 ? j : a3;
    if (r == 3) out[(int64_t)(o >> 2) * ld + i] = make_int4(a0, a1, a2, a3);
  }
  // pad the last partial quad with the atom itself (a valid, masked address)
  __device__ __forceinline__ void finish(int32_t o) {
    if (o & 3) {
      for (int32_t k = o; k & 3; ++k) put(k, i);
    }
  }
};

// The far segment of a split row, written from the back: the k-th far entry
// sits at slot cap4 - 1 - k; a quad is stored when its lowest slot is filled.
struct FarWriter {
  int4* out;
  int64_t ld;
  int32_t i, cap4;
  int32_t a0, a1, a2, a3;
  __device__ __forceinline__ void put(int32_t k, int32_t j) {
    const int32_t o = cap4 - 1 - k;
    const int r = o & 3;
    a0 = r == 0 ? j : a0;
    a1 = r == 1 ? j : a1;
    a2 = r == 2 ? j : a2;
    a3 = r == 3 ? j : a3;
    if (r == 0) out[(int64_t)(o >> 2) * ld + i] = make_int4(a0, a1, a2, a3);
  }
  // pad down to the quad boundary with the atom itself
  __device__ __forceinline__ void finish(int32_t k) {
    for (; (cap4 - k) & 3; ++k) put(k, i);
  }
};

// Thread-per-atom list build (the production builder).  With the cell-ordered
// store the 32 atoms of a warp sit in one or two cells, so they walk the
// same (2H+1)^2 stencil runs and their loop bounds barely diverge; candidate
// positions stream from the cell-ordered copy.  Tiered rows take two passes
// over the candidates: the first counts per tier, the second writes each
// entry at its tier's cursor.  Counters and cursors are eight 16-bit fields
// packed in two 64-bit registers (no dynamically indexed arrays, no local
// memory); each thread's writes fill its quads front to back within
// microseconds, so L2 merges the sectors before they leave.
template <typename F>
__device__ __forceinline__ void scan_stencil(const Cells& C, int H, int cid, F&& f) {
  const Stencil g = C.g;
  const int c2 = cid % g.g2, c1 = (cid / g.g2) % g.g1, c0 = cid / (g.g1 * g.g2);
  const int zlo = c2 - H > 0 ? c2 - H : 0, zhi = c2 + H < g.g2 ? c2 + H : g.g2 - 1;
  for (int ca = c0 - H; ca <= c0 + H; ++ca) {
    if (ca < 0 || ca >= g.g0) continue;
    for (int cb = c1 - H; cb <= c1 + H; ++cb) {
      if (cb < 0 || cb >= g.g1) continue;
      const int base = (ca * g.g1 + cb) * g.g2;
      const int32_t e = __ldg(C.cell_start + base + zhi + 1);
#pragma unroll 4
      for (int32_t k = __ldg(C.cell_start + base + zlo); k < e; ++k) f(k);
    }
  }
}

// The same walk with the distance test of NC consecutive candidates
// evaluated together (their 3 NC position loads in flight at once) and the
// accepted ones handled afterwards in candidate order.
template <int NC, typename R, typename F>
__device__ __forceinline__ void scan_stencil_chunked(const Cells& C, int H, int cid, R&& rsqb, F&& hit) {
  const Stencil g = C.g;
  const int c2 = cid % g.g2, c1 = (cid / g.g2) % g.g1, c0 = cid / (g.g1 * g.g2);
  const int zlo = c2 - H > 0 ? c2 - H : 0, zhi = c2 + H < g.g2 ? c2 + H : g.g2 - 1;
  for (int ca = c0 - H; ca <= c0 + H; ++ca) {
    if (ca < 0 || ca >= g.g0) continue;
    for (int cb = c1 - H; cb <= c1 + H; ++cb) {
      if (cb < 0 || cb >= g.g1) continue;
      const int base = (ca * g.g1 + cb) * g.g2;
      const int32_t e = __ldg(C.cell_start + base + zhi + 1);
      int32_t k = __ldg(C.cell_start + base + zlo);
      for (; k + NC <= e; k += NC) {
        long long b[NC];
#pragma unroll
        for (int u = 0; u < NC; ++u) b[u] = rsqb(k + u);
#pragma unroll
        for (int u = 0; u < NC; ++u) hit(k + u, b[u]);
      }
      for (; k < e; ++k) hit(k, rsqb(k));
    }
  }
}

template <bool TIERED, int CHUNK = 0>
__global__ void __launch_bounds__(128) k_build_thread(
    const double* __restrict__ pos, int64_t ld, int32_t n_local, Cells C, int H, double rsq_max, int half,
    Tiers T, int32_t cap, int32_t* __restrict__ nbr, int64_t ld_nbr, int32_t* __restrict__ tcnt,
    int32_t* __restrict__ nnbr, int64_t* __restrict__ st) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_local) return;
  // warps walk the stencil in cell order (coherent z-runs) whatever the order
  // of the rows they write
  const int32_t i = C.order ? C.order[t] : t;
  long long r2b[kMaxTiers];
#pragma unroll
  for (int q = 0; q < kMaxTiers; ++q) r2b[q] = __double_as_longlong(T.r2[q]);
  const long long maxb = __double_as_longlong(rsq_max);
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int cid = C.cell_of[i];
  if (cid < 0) {  // rejected by binning (status already raised): an empty row, never chased
    nnbr[i] = 0;
    if (TIERED) tcnt[i] = 0;
    return;
  }
  auto rsq_bits = [&](int32_t k) {
    return __double_as_longlong(rsq_ref(sub_rn(xi, __ldg(C.cp + k)), sub_rn(yi, __ldg(C.cp + C.ld_cp + k)),
                                        sub_rn(zi, __ldg(C.cp + 2 * C.ld_cp + k))));
  };
  if (!TIERED) {
    QuadWriter w{reinterpret_cast<int4*>(nbr), ld_nbr, i, i, i, i, i};
    int32_t cnt = 0;
    scan_stencil(C, H, cid, [&](int32_t k) {
      const int32_t j = __ldg(C.cell_atoms + k);
      if (half ? !(j >= n_local || j > i) : (j == i)) return;
      if (rsq_bits(k) < maxb) {
        if (cnt < cap) w.put(cnt, j);
        ++cnt;
      }
    });
    nnbr[i] = cnt;
    if (cnt > cap) {
      need_capacity(st, cnt);
      return;
    }
    w.finish(cnt);
    return;
  }
  // split rows, one pass: "near" entries (rsq < near_rsq) from the front of the
  // row ascending, "far" entries from the back descending — both as whole quads
  const int32_t cap4 = (cap + 3) & ~3;
  const long long nearb = r2b[0];
  QuadWriter w{reinterpret_cast<int4*>(nbr), ld_nbr, i, i, i, i, i};
  FarWriter fw{reinterpret_cast<int4*>(nbr), ld_nbr, i, cap4, i, i, i, i};
  int32_t nn = 0, nf = 0;
  auto hit = [&](int32_t k, long long b) {
    if (b < maxb) {
      const int32_t j = __ldg(C.cell_atoms + k);
      if (j == i) return;
      if (b < nearb) {
        if (((nn + 4) & ~3) + ((nf + 3) & ~3) <= cap4) w.put(nn, j);
        ++nn;
      } else {
        if (((nn + 3) & ~3) + ((nf + 4) & ~3) <= cap4) fw.put(nf, j);
        ++nf;
      }
    }
  };
  if (CHUNK > 0)
    scan_stencil_chunked<(CHUNK > 0 ? CHUNK : 1)>(C, H, cid, rsq_bits, hit);
  else
    scan_stencil(C, H, cid, [&](int32_t k) { hit(k, rsq_bits(k)); });
  const int32_t need = ((nn + 3) & ~3) + ((nf + 3) & ~3);
  nnbr[i] = nn + nf;
  tcnt[i] = nn;
  if (need > cap4) {
    need_capacity(st, need);
    return;
  }
  w.finish(nn);
  fw.finish(nf);
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

// ---------------------------------------------------------------------------
// Brick staging for the shared-memory step kernel (tmd_step_lj_brick).
// Locals are sorted brick-major (tmd_brick_sort): brick b = 4 x 4 x 4 interior
// cells of the r/2 grid.  Its staging set is every atom of the 8 x 8 columns
// around it over the z-run [4 bz - 2, min(4 bz + 4, d2) + 2) -- a superset of
// the 5^3 stencils of its atoms.  Column c = (x - 4 bx + 2) * 8 + (y - 4 by + 2)
// is one contiguous range of cell_atoms; the staged copy of cell_atoms[k] sits
// at stg_off[b][c] + (k - stg_start[b][c]).  List entries of the brick's atoms
// are these uint16 staging indices.
// ---------------------------------------------------------------------------
struct BrickGrid {
  int d[3];   // interior cells per dimension
  int nb[3];  // bricks per dimension
  int H;      // ghost shell layers (2)
  Stencil g;  // grid dims incl. the shell
};

__device__ __forceinline__ void brick_coords(const BrickGrid& B, int b, int& bx, int& by, int& bz) {
  bz = b % B.nb[2];
  by = (b / B.nb[2]) % B.nb[1];
  bx = b / (B.nb[1] * B.nb[2]);
}

// one warp per brick: column ranges and their exclusive prefix
__global__ void k_brick_meta(BrickGrid B, int32_t n_bricks, const int32_t* __restrict__ cell_start,
                             int32_t* __restrict__ stg_start, int32_t* __restrict__ stg_off,
                             int32_t* __restrict__ max_stage) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= n_bricks) return;
  int bx, by, bz;
  brick_coords(B, b, bx, by, bz);
  const int zlo = 4 * bz - 2, zhi = min(4 * bz + 4, B.d[2]) + 2;  // interior coords, [zlo, zhi)
  const int xhi = min(4 * bx + 4, B.d[0]) + 2, yhi = min(4 * by + 4, B.d[1]) + 2;
  int32_t st[2], len[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    const int x = 4 * bx - 2 + (c >> 3), y = 4 * by - 2 + (c & 7);
    st[h] = 0;
    len[h] = 0;
    if (x < xhi && y < yhi) {
      const int base = ((x + B.H) * B.g.g1 + (y + B.H)) * B.g.g2;
      st[h] = cell_start[base + zlo + B.H];
      len[h] = cell_start[base + zhi + B.H] - st[h];
    }
  }
  // warp-inclusive scans of the two halves, the second offset by the first's total
  int32_t inc0 = len[0], inc1 = len[1];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t t0 = __shfl_up_sync(0xffffffffu, inc0, o);
    const int32_t t1 = __shfl_up_sync(0xffffffffu, inc1, o);
    if (lane >= o) {
      inc0 += t0;
      inc1 += t1;
    }
  }
  const int32_t tot0 = __shfl_sync(0xffffffffu, inc0, 31);
  const int32_t tot = tot0 + __shfl_sync(0xffffffffu, inc1, 31);
  stg_start[(int64_t)b * 64 + lane] = st[0];
  stg_start[(int64_t)b * 64 + 32 + lane] = st[1];
  stg_off[(int64_t)b * 65 + lane] = inc0 - len[0];
  stg_off[(int64_t)b * 65 + 32 + lane] = tot0 + inc1 - len[1];
  if (lane == 0) {
    stg_off[(int64_t)b * 65 + 64] = tot;
    atomicMax(max_stage, tot);
  }
}

// Eight uint16 entries packed in registers and stored as one 16-byte uint4:
// octet q of atom i at out[q * ld + i].
struct OctWriter {
  uint4* out;
  int64_t ld;
  int32_t i;
  uint32_t a0, a1, a2, a3;
  __device__ __forceinline__ void set(int r, uint32_t v) {
    const uint32_t sh = (r & 1) * 16, keep = ~(0xFFFFu << sh), val = v << sh;
    const int q = r >> 1;
    a0 = q == 0 ? ((a0 & keep) | val) : a0;
    a1 = q == 1 ? ((a1 & keep) | val) : a1;
    a2 = q == 2 ? ((a2 & keep) | val) : a2;
    a3 = q == 3 ? ((a3 & keep) | val) : a3;
  }
  __device__ __forceinline__ void store(int32_t q) { out[(int64_t)q * ld + i] = make_uint4(a0, a1, a2, a3); }
};

// FAR: the k-th entry sits at slot cap8 - 1 - k and an octet is stored when its
// lowest slot is filled; front: slot k, stored when its highest slot is filled
template <bool FAR>
__device__ __forceinline__ void oct_put(OctWriter& w, int32_t cap8, int32_t k, uint32_t v) {
  const int32_t o = FAR ? cap8 - 1 - k : k;
  const int r = o & 7;
  w.set(r, v);
  if (FAR ? (r == 0) : (r == 7)) w.store(o >> 3);
}

// pad with staging index 0 (a valid address, masked by the counts)
template <bool FAR>
__device__ __forceinline__ void oct_finish(OctWriter& w, int32_t cap8, int32_t k) {
  if (FAR) {
    for (; (cap8 - k) & 7; ++k) oct_put<true>(w, cap8, k, 0);
  } else {
    for (; k & 7; ++k) oct_put<false>(w, cap8, k, 0);
  }
}

// Split rows of uint16 staging indices, one block per brick: the brick's
// staging set (current positions) and the staging index of every cell start
// of its 8 x 8 columns go to shared memory, then each thread walks its atom's
// 5^3 stencil as 25 runs of staging indices with the same membership test and
// near/far split as k_build_thread<true> (reference-order rsq, bit-exact).
constexpr int kBuildBrickThreads = 160;

__global__ void __launch_bounds__(kBuildBrickThreads) k_build_brick(
    const double* __restrict__ pos, int64_t ld, const int32_t* __restrict__ key_start,
    const int32_t* __restrict__ cell_of, const int32_t* __restrict__ cell_start,
    const int32_t* __restrict__ cell_atoms, BrickGrid B, const int32_t* __restrict__ stg_start,
    const int32_t* __restrict__ stg_off, double near_rsq, double rsq_max, int32_t cap, uint16_t* __restrict__ nbr,
    int64_t ld_nbr, int32_t* __restrict__ nnear, int32_t* __restrict__ nnbr, int64_t* __restrict__ st,
    int32_t max_stage) {
  extern __shared__ double stage[];
  double* sx = stage;
  double* sy = stage + max_stage;
  double* sz = stage + 2 * max_stage;
  __shared__ int32_t s_off[65], s_st[64], s_key[65], s_cell[64 * 9];
  const int b = blockIdx.x;
  const int32_t a0 = key_start[(int64_t)b * 64], a1 = key_start[(int64_t)(b + 1) * 64];
  if (a1 == a0) return;
  if (threadIdx.x < 65) {
    s_off[threadIdx.x] = stg_off[(int64_t)b * 65 + threadIdx.x];
    s_key[threadIdx.x] = key_start[(int64_t)b * 64 + threadIdx.x];
  }
  if (threadIdx.x < 64) s_st[threadIdx.x] = stg_start[(int64_t)b * 64 + threadIdx.x];
  __syncthreads();
  int bx, by, bz;
  brick_coords(B, b, bx, by, bz);
  const int zlo = 4 * bz - 2, nz = min(4 * bz + 4, B.d[2]) + 2 - zlo;  // staging z-run (interior coords)
  const int xhi = min(4 * bx + 4, B.d[0]) + 2, yhi = min(4 * by + 4, B.d[1]) + 2;
  for (int t = threadIdx.x; t < 64 * 9; t += blockDim.x) {
    const int c = t / 9, dz = t - 9 * (t / 9);
    const int x = 4 * bx - 2 + (c >> 3), y = 4 * by - 2 + (c & 7);
    int32_t v = s_off[c];
    if (dz <= nz && x < xhi && y < yhi)
      v += cell_start[((x + B.H) * B.g.g1 + (y + B.H)) * B.g.g2 + zlo + dz + B.H] - s_st[c];
    s_cell[t] = v;
  }
  stage_positions(pos, ld, cell_atoms, s_off, s_st, sx, sy, sz);
  __syncthreads();
  const long long maxb = __double_as_longlong(rsq_max), nearb = __double_as_longlong(near_rsq);
  const int32_t cap8 = (cap + 7) & ~7;
  for (int32_t i = a0 + threadIdx.x; i < a1; i += blockDim.x) {
    // i's cell in the brick: the last key whose first local is <= i
    int lo = 0, hi = 64;
#pragma unroll
    for (int it = 0; it < 6; ++it) {
      const int mid = (lo + hi) >> 1;
      if (s_key[mid] <= i) lo = mid; else hi = mid;
    }
    const int lx = lo >> 4, ly = (lo >> 2) & 3, lz = lo & 3;
    // the sort key and the build grid must agree on i's cell
    const int cid = ((4 * bx + lx + B.H) * B.g.g1 + (4 * by + ly + B.H)) * B.g.g2 + 4 * bz + lz + B.H;
    if (cell_of[i] != cid) {
      raise_status(st, TMD_PROTOCOL, (unsigned long long)i);
      nnbr[i] = 0;
      nnear[i] = 0;
      continue;
    }
    const int32_t own = s_cell[((lx + 2) * 8 + (ly + 2)) * 9 + lz + 2] + (i - s_key[lo]);
    const double xi = sx[own], yi = sy[own], zi = sz[own];
    OctWriter fw{reinterpret_cast<uint4*>(nbr), ld_nbr, i, 0u, 0u, 0u, 0u};
    OctWriter bw{reinterpret_cast<uint4*>(nbr), ld_nbr, i, 0u, 0u, 0u, 0u};
    int32_t nn = 0, nf = 0;
    for (int dx = 0; dx < 5; ++dx) {
      for (int dy = 0; dy < 5; ++dy) {
        const int row = ((lx + dx) * 8 + (ly + dy)) * 9 + lz;
        const int32_t s1 = s_cell[row + 5];
        for (int32_t s = s_cell[row]; s < s1; ++s) {
          const long long bb =
              __double_as_longlong(rsq_ref(sub_rn(xi, sx[s]), sub_rn(yi, sy[s]), sub_rn(zi, sz[s])));
          if (bb < maxb && s != own) {
            if (bb < nearb) {
              if (((nn + 8) & ~7) + ((nf + 7) & ~7) <= cap8) oct_put<false>(fw, cap8, nn, (uint32_t)s);
              ++nn;
            } else {
              if (((nn + 7) & ~7) + ((nf + 8) & ~7) <= cap8) oct_put<true>(bw, cap8, nf, (uint32_t)s);
              ++nf;
            }
          }
        }
      }
    }
    const int32_t need = ((nn + 7) & ~7) + ((nf + 7) & ~7);
    nnbr[i] = nn + nf;
    nnear[i] = nn;
    if (need > cap8) {
      need_capacity(st, need);
      continue;
    }
    oct_finish<false>(fw, cap8, nn);
    oct_finish<true>(bw, cap8, nf);
  }
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
  C.order = nullptr;
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
  const int B = 128;
  // builder variant: candidates evaluated in chunks of TMD_BUILD_CHUNK (4 by
  // default; 0 = one at a time)
  static int chunk = [] {
    const char* e = getenv("TMD_BUILD_CHUNK");
    return e ? atoi(e) : 4;
  }();
  if (TIERED && chunk >= 8)
    k_build_thread<TIERED, 8><<<grid_for(n_local, B), B, 0, s>>>(d_pos, ld, n_local, C, H, rsq_max, half, T, cap,
                                                                 d_nbr, ld_nbr, d_tcnt, d_nnbr, d_status);
  else if (TIERED && chunk >= 2)
    k_build_thread<TIERED, 4><<<grid_for(n_local, B), B, 0, s>>>(d_pos, ld, n_local, C, H, rsq_max, half, T, cap,
                                                                 d_nbr, ld_nbr, d_tcnt, d_nnbr, d_status);
  else
    k_build_thread<TIERED><<<grid_for(n_local, B), B, 0, s>>>(d_pos, ld, n_local, C, H, rsq_max, half, T, cap,
                                                             d_nbr, ld_nbr, d_tcnt, d_nnbr, d_status);
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

extern "C" int tmd_build_lists_split(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_cell_of,
                                     const int32_t* d_cell_start, const int32_t* d_cell_atoms,
                                     const double* d_cell_pos, int64_t ld_cp, const int32_t* h_dims, int32_t shell,
                                     double near_rsq, double rsq_max, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                                     int32_t* d_nnear, int32_t* d_nnbr, const int32_t* d_order, int64_t* d_status,
                                     void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!h_dims || !d_cell_pos || cap < 0 || ld_nbr < n_local || shell < 1 || !(near_rsq <= rsq_max))
    return TMD_ERR_ARG;
  Tiers T{};
  T.r2[0] = near_rsq;
  T.nt = 1;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims, shell);
  C.order = d_order;
  return launch_build<true>(d_pos, ld, n_local, C, shell, rsq_max, 0, T, cap, d_nbr, ld_nbr, d_nnear, d_nnbr,
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

static bool brick_grid(const int32_t* h_dims, int shell, BrickGrid* B) {
  for (int d = 0; d < 3; ++d) {
    if (h_dims[d] < 1) return false;
    B->d[d] = h_dims[d];
    B->nb[d] = (h_dims[d] + 3) / 4;
  }
  B->H = shell;
  B->g = Stencil{h_dims[0] + 2 * shell, h_dims[1] + 2 * shell, h_dims[2] + 2 * shell};
  return shell == 2;
}

extern "C" int tmd_brick_meta(const int32_t* d_cell_start, const int32_t* h_dims, int32_t shell,
                              int32_t* d_stg_start, int32_t* d_stg_off, int32_t* d_max_stage, void* stream) {
  BrickGrid B;
  if (!h_dims || !brick_grid(h_dims, shell, &B)) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  const int32_t n_bricks = B.nb[0] * B.nb[1] * B.nb[2];
  TMD_CUDA_TRY(cudaMemsetAsync(d_max_stage, 0, sizeof(int32_t), s), "brick_meta");
  k_brick_meta<<<(n_bricks + 3) / 4, 128, 0, s>>>(B, n_bricks, d_cell_start, d_stg_start, d_stg_off, d_max_stage);
  TMD_LAUNCH_CHECK("brick_meta");
  return TMD_OK;
}

extern "C" int tmd_build_lists_brick(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_cell_of,
                                     const int32_t* d_cell_start, const int32_t* d_cell_atoms,
                                     const int32_t* d_key_start, int32_t max_stage, const int32_t* h_dims,
                                     int32_t shell, const int32_t* d_stg_start, const int32_t* d_stg_off,
                                     double near_rsq, double rsq_max, int32_t cap, uint16_t* d_nbr, int64_t ld_nbr,
                                     int32_t* d_nnear, int32_t* d_nnbr, int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  BrickGrid B;
  if (!h_dims || !d_key_start || cap < 0 || ld_nbr < n_local || !(near_rsq <= rsq_max) ||
      !brick_grid(h_dims, shell, &B) || max_stage < 1 || max_stage > 65536)
    return TMD_ERR_ARG;
  const size_t smem = sizeof(double) * 3 * (size_t)max_stage;
  if (smem > 200 * 1024) return TMD_ERR_ARG;
  static bool attr = false;
  if (!attr) {
    TMD_CUDA_TRY(cudaFuncSetAttribute(k_build_brick, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                 "build_lists_brick smem attribute");
    attr = true;
  }
  const int32_t n_bricks = B.nb[0] * B.nb[1] * B.nb[2];
  k_build_brick<<<n_bricks, kBuildBrickThreads, smem, as_stream(stream)>>>(
      d_pos, ld, d_key_start, d_cell_of, d_cell_start, d_cell_atoms, B, d_stg_start, d_stg_off, near_rsq, rsq_max,
      cap, d_nbr, ld_nbr, d_nnear, d_nnbr, d_status, max_stage);
  TMD_LAUNCH_CHECK("build_lists_brick");
  return TMD_OK;
}
