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
//  * reference order (tmd_build_lists, thread per atom): rows identical slot
//    for slot to the reference; the rsq predicate is evaluated in the
//    reference's operation order, so membership is bit-exact.
//  * split rows (tmd_build_lists_split, production, warp per cell of the r/2
//    grid): same membership; pairs within cutoff + margin at the front of
//    the row, the rest at the back (the step kernel's exact pruning).
#include <cmath>

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

__global__ void __launch_bounds__(128) k_build_thread(
    const double* __restrict__ pos, int64_t ld, int32_t n_local, Cells C, int H, double rsq_max, int half,
    int32_t cap, int32_t* __restrict__ nbr, int64_t ld_nbr, int32_t* __restrict__ nnbr, int64_t* __restrict__ st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  const long long maxb = __double_as_longlong(rsq_max);
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int cid = C.cell_of[i];
  if (cid < 0) {  // rejected by binning (status already raised): an empty row, never chased
    nnbr[i] = 0;
    return;
  }
  // non-negative doubles order like their bit patterns
  auto rsq_bits = [&](int32_t k) {
    return __double_as_longlong(rsq_ref(sub_rn(xi, __ldg(C.cp + k)), sub_rn(yi, __ldg(C.cp + C.ld_cp + k)),
                                        sub_rn(zi, __ldg(C.cp + 2 * C.ld_cp + k))));
  };
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
}

// ---------------------------------------------------------------------------
// Production split-row builder: one warp per cell of the r/2 grid.
//
// All atoms of a cell share one (2H+1)^2-column stencil; its 25 z-runs are
// contiguous ranges of the cell-ordered positions.  The warp concatenates the
// runs (a warp scan of their lengths) and walks the candidates 32 at a time,
// one per lane, so every lane does useful work whatever the run lengths; the
// next 32 candidates are fetched while the current ones are tested.  Each
// candidate is tested against every atom of the cell (kCellAtoms per pass).
//
// The distance test runs in FP32 on a float4 copy of the cell-ordered
// positions relative to the grid origin, with a proven error bound delta
// (host: 4e-6 X + 5e-5 for coordinates |x - lo| <= X): a candidate whose FP32
// rsq lies within delta of r^2 or of near_rsq is decided by the reference's
// FP64 rsq in its own operation order (neighbor.py:127-139), so membership
// and the near/far split are exactly the FP64 ones.  Hits are compacted with
// ballots: near pairs fill the row from the front, far pairs from the back;
// order inside a segment is stencil-run order.  Rows are written in the
// atoms' own numbering (brick-major on the production path).
// ---------------------------------------------------------------------------
constexpr int kCellAtoms = 4;
constexpr int kBuildWarps = 4;

struct SplitTest {
  float hit_lo, hit_hi;    // rsq32 < hit_lo: inside r; >= hit_hi: outside; else FP64
  float near_lo, near_hi;  // same around near_rsq
  double rsq_max, near_rsq;
};


__global__ void k_cell_pos4(const double* __restrict__ cp, int64_t ld_cp, int32_t n, double lo0, double lo1,
                            double lo2, float4* __restrict__ out) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  out[k] = make_float4((float)(cp[k] - lo0), (float)(cp[ld_cp + k] - lo1), (float)(cp[2 * ld_cp + k] - lo2), 0.f);
}

__global__ void __launch_bounds__(32 * kBuildWarps, 6) k_build_cells(
    int32_t n_local, Cells C, const float4* __restrict__ cp4, int H, int32_t n_cells, SplitTest T, int32_t cap4,
    int32_t* __restrict__ nbr, int64_t ld_nbr, int32_t* __restrict__ nnear, int32_t* __restrict__ nnbr,
    int64_t* __restrict__ st) {
  // the rows of the cell's atoms are assembled here and leave as whole int4
  // quads (scattered 4-byte stores into the list cost L2 partial-sector
  // read-modify-writes): kBuildWarps x kCellAtoms rows of cap4 slots
  extern __shared__ __align__(16) int32_t s_rows[];
  const int lane = threadIdx.x & 31;
  const int32_t c = blockIdx.x * kBuildWarps + (threadIdx.x >> 5);
  if (c >= n_cells) return;
  const int32_t cs = __ldg(C.cell_start + c), ce = __ldg(C.cell_start + c + 1);
  // locals come first in a cell (ascending atom index, ghosts >= n_local)
  int32_t na = 0;
  for (int32_t k0 = cs; k0 < ce; k0 += 32) {
    const bool loc = k0 + lane < ce && __ldg(C.cell_atoms + k0 + lane) < n_local;
    na += __popc(__ballot_sync(0xffffffffu, loc));
  }
  if (na == 0) return;
  const Stencil g = C.g;
  const int c2 = c % g.g2, c1 = (c / g.g2) % g.g1, c0 = c / (g.g1 * g.g2);
  const int zlo = c2 - H > 0 ? c2 - H : 0, zhi = c2 + H < g.g2 ? c2 + H : g.g2 - 1;
  const int W = 2 * H + 1;
  // lane r < W^2: run r = column (c0 + r / W - H, c1 + r % W - H) over [zlo, zhi]
  int32_t rs = 0, rl = 0;
  if (lane < W * W) {
    const int ca = c0 + lane / W - H, cb = c1 + lane % W - H;
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
  const int32_t excl = incl - rl;
  const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const unsigned lt = (1u << lane) - 1u;
  // cell-order index of candidate t0 + lane (cs beyond the last candidate):
  // the last run r < W^2 with excl_r <= t (excl is non-decreasing over
  // lanes); five fixed steps, so every lane takes part in every shuffle
  auto cand = [&](int32_t t0) {
    const int32_t t = t0 + lane;
    int lo = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int mid = lo + step;
      const int32_t e = __shfl_sync(0xffffffffu, excl, mid < 32 ? mid : 31);
      if (mid < W * W && e <= t) lo = mid;
    }
    const int32_t k = __shfl_sync(0xffffffffu, rs, lo) + (t - __shfl_sync(0xffffffffu, excl, lo));
    return t < total ? k : cs;
  };
  for (int32_t a0 = 0; a0 < na; a0 += kCellAtoms) {
    const int32_t nb = na - a0 < kCellAtoms ? na - a0 : kCellAtoms;
    int32_t* rows = s_rows + (size_t)(threadIdx.x >> 5) * kCellAtoms * cap4;
    int32_t ia[kCellAtoms], nn[kCellAtoms], nf[kCellAtoms];
    float xa[kCellAtoms], ya[kCellAtoms], za[kCellAtoms];
#pragma unroll
    for (int a = 0; a < kCellAtoms; ++a) {
      const int32_t k = cs + a0 + (a < nb ? a : 0);
      ia[a] = __ldg(C.cell_atoms + k);
      const float4 q = __ldg(cp4 + k);
      xa[a] = q.x;
      ya[a] = q.y;
      za[a] = q.z;
      nn[a] = 0;
      nf[a] = 0;
    }
    int32_t kk = cand(0);
    float4 q = __ldg(cp4 + kk);
    int32_t j = __ldg(C.cell_atoms + kk);
    for (int32_t t0 = 0; t0 < total; t0 += 32) {
      const bool valid = t0 + lane < total;
      const int32_t k_cur = kk;
      // prefetch the next 32 candidates
      int32_t kn = cs;
      float4 qn = q;
      int32_t jn = j;
      if (t0 + 32 < total) {
        kn = cand(t0 + 32);
        qn = __ldg(cp4 + kn);
        jn = __ldg(C.cell_atoms + kn);
      }
#pragma unroll
      for (int a = 0; a < kCellAtoms; ++a) {
        if (a >= nb) break;  // warp-uniform
        const float dx = xa[a] - q.x, dy = ya[a] - q.y, dz = za[a] - q.z;
        const float r32 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        bool hit = r32 < T.hit_lo, near = r32 < T.near_lo;
        const bool other = valid && j != ia[a];
        if (other && ((r32 < T.hit_hi) != hit || (r32 < T.near_hi) != near)) {
          // within the FP32 error band of a threshold (rare): the reference's FP64 rsq decides
          const int32_t ka = cs + a0 + a;
          const double rsq = rsq_ref(sub_rn(__ldg(C.cp + ka), __ldg(C.cp + k_cur)),
                                     sub_rn(__ldg(C.cp + C.ld_cp + ka), __ldg(C.cp + C.ld_cp + k_cur)),
                                     sub_rn(__ldg(C.cp + 2 * C.ld_cp + ka), __ldg(C.cp + 2 * C.ld_cp + k_cur)));
          hit = rsq < T.rsq_max;
          near = rsq < T.near_rsq;
        }
        hit = hit && other;
        near = near && hit;
        const bool far = hit && !near;
        const unsigned bn = __ballot_sync(0xffffffffu, near);
        const unsigned bf = __ballot_sync(0xffffffffu, far);
        const int32_t sn = nn[a] + __popc(bn & lt);
        const int32_t sf = cap4 - 1 - (nf[a] + __popc(bf & lt));
        int32_t* row = rows + a * cap4;
        if (near && sn < cap4) row[sn] = j;
        if (far && sf >= 0) row[sf] = j;
        nn[a] += __popc(bn);
        nf[a] += __popc(bf);
      }
      kk = kn;
      q = qn;
      j = jn;
    }
#pragma unroll
    for (int a = 0; a < kCellAtoms; ++a) {
      if (a >= nb) break;
      const int32_t need = ((nn[a] + 3) & ~3) + ((nf[a] + 3) & ~3);
      if (need > cap4) {
        if (lane == 0) {
          need_capacity(st, need);
          nnbr[ia[a]] = nn[a] + nf[a];
          nnear[ia[a]] = nn[a];
        }
        continue;
      }
      // pad the partial quads of both segments with the atom itself (a valid,
      // masked address), then store the row's used quads as int4s
      int32_t* row = rows + a * cap4;
      const int32_t qn = (nn[a] + 3) >> 2, qf = (nf[a] + 3) >> 2;
      if (lane < 3) {
        const int32_t kq = nn[a] + lane;
        if (kq < 4 * qn) row[kq] = ia[a];
      } else if (lane < 6) {
        const int32_t kf = cap4 - 1 - (nf[a] + lane - 3);
        if (kf >= cap4 - 4 * qf) row[kf] = ia[a];
      }
      __syncwarp();
      int4* out = reinterpret_cast<int4*>(nbr);
      for (int32_t q = lane; q < qn + qf; q += 32) {
        const int32_t qq = q < qn ? q : (cap4 >> 2) - qf + (q - qn);
        out[(int64_t)qq * ld_nbr + ia[a]] = *reinterpret_cast<const int4*>(row + 4 * qq);
      }
      if (lane == 0) {
        nnbr[ia[a]] = nn[a] + nf[a];
        nnear[ia[a]] = nn[a];
      }
    }
    __syncwarp();  // the rows are reused by the next group of the cell's atoms
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

extern "C" int tmd_build_lists(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_cell_of,
                               const int32_t* d_cell_start, const int32_t* d_cell_atoms,
                               const double* d_cell_pos, int64_t ld_cp, const int32_t* h_dims,
                               double rsq_max, int32_t half, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                               int32_t* d_nnbr, int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!h_dims || !d_cell_pos || cap < 0 || ld_nbr < n_local) return TMD_ERR_ARG;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims, 1);
  k_build_thread<<<grid_for(n_local, 128), 128, 0, as_stream(stream)>>>(d_pos, ld, n_local, C, 1, rsq_max, half,
                                                                         cap, d_nbr, ld_nbr, d_nnbr, d_status);
  TMD_LAUNCH_CHECK("build_lists");
  return TMD_OK;
}

extern "C" int tmd_build_lists_split(const double* d_pos, int64_t ld, int32_t n_local, int32_t n_total,
                                     const int32_t* d_cell_of, const int32_t* d_cell_start,
                                     const int32_t* d_cell_atoms, const double* d_cell_pos, int64_t ld_cp,
                                     const double* h_lo, double extent_max,
                                     const int32_t* h_dims, int32_t shell, double near_rsq, double rsq_max,
                                     int32_t cap, int32_t* d_nbr, int64_t ld_nbr, int32_t* d_nnear, int32_t* d_nnbr,
                                     int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!h_dims || !h_lo || !d_cell_pos || cap < 0 || ld_nbr < n_local || n_total < n_local || ld_cp < n_total ||
      shell < 1 || shell > 2 ||
      !(near_rsq <= rsq_max) || !(extent_max > 0.0))
    return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims, shell);
  const int64_t n_cells = (int64_t)C.g.g0 * C.g.g1 * C.g.g2;
  // FP32 error bound of rsq for |x - lo| <= X (see the kernel comment)
  const double X = extent_max + 4.0 * sqrt(rsq_max);
  const double delta = 4e-6 * X + 5e-5;
  SplitTest T;
  T.rsq_max = rsq_max;
  T.near_rsq = near_rsq;
  T.hit_lo = nextafterf((float)(rsq_max - delta), 0.f);
  T.hit_hi = nextafterf((float)(rsq_max + delta), 1e30f);
  T.near_lo = nextafterf((float)(near_rsq - delta), 0.f);
  T.near_hi = nextafterf((float)(near_rsq + delta), 1e30f);
  keep_pool_memory();
  float4* cp4 = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cp4), sizeof(float4) * (size_t)n_total, s),
               "build_lists_split scratch");
  k_cell_pos4<<<grid_for(n_total, 256), 256, 0, s>>>(d_cell_pos, ld_cp, n_total, h_lo[0], h_lo[1], h_lo[2], cp4);
  TMD_LAUNCH_CHECK("cell_pos4");
  const int blocks = (int)((n_cells + kBuildWarps - 1) / kBuildWarps);
  const int32_t cap4 = (cap + 3) & ~3;
  const size_t smem = sizeof(int32_t) * (size_t)kBuildWarps * kCellAtoms * cap4;
  if (smem > 160 * 1024) return TMD_ERR_ARG;  // rows of > 2560 slots
  if (smem > 48 * 1024) {
    TMD_CUDA_TRY(cudaFuncSetAttribute(k_build_cells, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024),
                 "build_lists_split smem attribute");
  }
  k_build_cells<<<blocks, 32 * kBuildWarps, smem, s>>>(n_local, C, cp4, shell, (int32_t)n_cells, T, cap4, d_nbr,
                                                       ld_nbr, d_nnear, d_nnbr, d_status);
  TMD_LAUNCH_CHECK("build_lists_split");
  TMD_CUDA_TRY(cudaFreeAsync(cp4, s), "build_lists_split scratch");
  return TMD_OK;
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
