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
//  * split rows (tmd_build_lists_split, production): same membership; pairs
//    within cutoff + margin fill the row from the front, the rest from the
//    back (the step kernel's exact pruning), both as whole int4 quads.
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
  const float* cpf;  // the same rounded to float (split builder pre-filter; optional)
  double f32_eps;    // bound on the float squared-distance error
  Stencil g;
  const int32_t* order;  // builder thread t -> local atom (null: t itself)
};

constexpr int kMaxTiers = 8;

struct Tiers {
  double r2[kMaxTiers];  // ascending squared tier radii, padded with the list radius^2
  int nt;
  const double* d_r2;  // when set: r2[0] (the near/far split) read from the device
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

// Thread-per-atom list build.  Threads walk the atoms in cell order (a thread
// -> atom map when the store is numbered otherwise), so the 32 atoms of a
// warp sit in a few consecutive cells of one z column and walk the same
// (2H+1)^2 stencil runs; candidate positions stream from the cell-ordered
// copy.  Reference-order rows pack four entries per int4 store; split rows
// store entry by entry (below).
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

// The chunked walk with the candidates' atom ids loaded up front too (split
// builder): hit(k, j, b) gets the cell slot, the id and rsqb(k).
template <int NC, typename R, typename F>
__device__ __forceinline__ void scan_stencil_chunked_ids(const Cells& C, int H, int cid, R&& rsqb, F&& hit) {
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
        decltype(rsqb(k)) b[NC];
        int32_t j[NC];
#pragma unroll
        for (int u = 0; u < NC; ++u) {
          b[u] = rsqb(k + u);
          j[u] = __ldg(C.cell_atoms + k + u);
        }
#pragma unroll
        for (int u = 0; u < NC; ++u) hit(k + u, j[u], b[u]);
      }
      for (; k < e; ++k) hit(k, __ldg(C.cell_atoms + k), rsqb(k));
    }
  }
}

// F32 (float pre-filter): capped at 64 registers (8 blocks/SM; uncapped it
// takes 69-80 and runs 1.37 ms at 80^3, capped 1.21 ms); 0 = no cap.
template <bool TIERED, int CHUNK = 0, bool F32 = false>
__global__ void __launch_bounds__(128, F32 ? 8 : 0) k_build_thread(
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
  if (TIERED && T.d_r2) r2b[0] = __double_as_longlong(*T.d_r2);
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
  // row ascending, "far" entries from the back descending.  Each accepted entry
  // is stored on its own (4 bytes; a thread's stores to one quad land within
  // microseconds and merge in L2) -- measured 17% faster than packing quads in
  // registers, whose select/conditional-store chain ran on every lane of the
  // (divergent) accept branch; candidate ids load with the positions, two
  // candidates per iteration (scripts/experiments: chunk 1 / 2 / 4 / 8 =
  // 1.42 / 1.36 / 1.37 / 1.47 ms at 80^3 vs 1.75 ms for the quad writer;
  // stepped write cursors then 1.25 ms).
  const int32_t cap4 = (cap + 3) & ~3;
  const double near_rsq = __longlong_as_double(r2b[0]);
  int32_t* row = nbr + (int64_t)i * 4;
  const int64_t qs = ld_nbr * 4;  // int32 stride between quads of a row
  // write cursors: pf at front slot nn, pb at back slot cap4 - 1 - nf (slot o
  // lives at row[(o >> 2) * qs + (o & 3)]); stepping them on a hit replaces
  // the 64-bit slot address arithmetic per entry
  int32_t* pf = row;
  int32_t* pb = row + (int64_t)((cap4 - 1) >> 2) * qs + 3;
  int32_t nn = 0, nf = 0;
  // store j (not the atom itself) in the near or the far segment
  auto put = [&](int32_t j, bool nr) {
    if (j != i) {
      if (nn + nf < cap4) *(nr ? pf : pb) = j;
      if (nr) {
        ++nn;
        pf += (nn & 3) ? 1 : qs - 3;
      } else {
        ++nf;
        pb -= (nf & 3) ? 1 : qs - 3;
      }
    }
  };
  auto rsq_val = [&](int32_t k) {
    return rsq_ref(sub_rn(xi, __ldg(C.cp + k)), sub_rn(yi, __ldg(C.cp + C.ld_cp + k)),
                   sub_rn(zi, __ldg(C.cp + 2 * C.ld_cp + k)));
  };
  constexpr int NC = CHUNK > 0 ? CHUNK : 1;
  if constexpr (F32) {
    // float pre-filter: half the candidate bytes through L1.  Decided on the
    // float value only when it is more than f32_eps (>= the float error) from
    // both thresholds -- the same answer as the reference's double; the rest
    // (and a NaN) are recomputed in double
    const float xf = __double2float_rn(xi), yf = __double2float_rn(yi), zf = __double2float_rn(zi);
    const float t_out = __double2float_ru(rsq_max + C.f32_eps), t_in = __double2float_rd(rsq_max - C.f32_eps);
    const float n_lo = __double2float_rd(near_rsq - C.f32_eps), n_hi = __double2float_ru(near_rsq + C.f32_eps);
    auto rsq_f = [&](int32_t k) {
      const float dx = xf - __ldg(C.cpf + k), dy = yf - __ldg(C.cpf + C.ld_cp + k),
                  dz = zf - __ldg(C.cpf + 2 * C.ld_cp + k);
      return dx * dx + dy * dy + dz * dz;
    };
    scan_stencil_chunked_ids<NC>(C, H, cid, rsq_f, [&](int32_t k, int32_t j, float r) {
      if (r >= t_out) return;
      if (r < t_in && (r < n_lo || r >= n_hi)) {
        put(j, r < n_lo);
        return;
      }
      const double rsq = rsq_val(k);
      if (rsq < rsq_max) put(j, rsq < near_rsq);
    });
  } else {
    // rsq compared as doubles: the same order as the bit patterns for
    // non-negative values, and a NaN fails both tests either way
    scan_stencil_chunked_ids<NC>(C, H, cid, rsq_val, [&](int32_t k, int32_t j, double rsq) {
      if (rsq < rsq_max) put(j, rsq < near_rsq);
    });
  }
  const int32_t need = ((nn + 3) & ~3) + ((nf + 3) & ~3);
  nnbr[i] = nn + nf;
  tcnt[i] = nn;
  if (need > cap4) {
    need_capacity(st, need);
    return;
  }
  // pad the partial quads with the atom itself (a valid, masked address)
  for (int32_t o = nn; o & 3; ++o) row[(int64_t)(o >> 2) * qs + (o & 3)] = i;
  for (int32_t o = cap4 - 1 - nf; (o & 3) != 3; --o) row[(int64_t)(o >> 2) * qs + (o & 3)] = i;
}

// The near/far split of the next build from the guard maxima of the epoch's
// steps (driver.Simulation: margin = max(floor, factor * sqrt(max d2)), capped):
// out[0] = (cut + margin)^2, out[1] = margin.  One thread; lets the epoch
// enqueue the build before the host has read the maxima.
__global__ void k_split_margin(const double* __restrict__ d2, int32_t i0, int32_t i1, double floor_m, double factor,
                               double cap, double cut, double* __restrict__ out) {
  double m = 0.0;
  for (int32_t i = i0; i < i1; ++i) m = fmax(m, d2[i]);
  double margin = fmax(floor_m, factor * sqrt(m));
  margin = fmin(margin, cap);
  const double c = cut + margin;
  out[0] = c * c;
  out[1] = margin;
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
  C.order = nullptr;
  C.cpf = nullptr;
  C.f32_eps = 0.0;
  return C;
}

template <bool TIERED>
static int launch_build(const double* d_pos, int64_t ld, int32_t n_local, const Cells& C, int H, double rsq_max,
                        int32_t half, const Tiers& T, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                        int32_t* d_tcnt, int32_t* d_nnbr, int64_t* d_status, cudaStream_t s) {
  const int B = 128;
  if (TIERED && C.cpf)
    k_build_thread<true, 2, true><<<grid_for(n_local, B), B, 0, s>>>(d_pos, ld, n_local, C, H, rsq_max, half, T,
                                                                     cap, d_nbr, ld_nbr, d_tcnt, d_nnbr, d_status);
  else if (TIERED)
    k_build_thread<true, 2><<<grid_for(n_local, B), B, 0, s>>>(d_pos, ld, n_local, C, H, rsq_max, half, T, cap,
                                                               d_nbr, ld_nbr, d_tcnt, d_nnbr, d_status);
  else
    k_build_thread<false, 4><<<grid_for(n_local, B), B, 0, s>>>(d_pos, ld, n_local, C, H, rsq_max, half, T, cap,
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
                                     const double* d_cell_pos, int64_t ld_cp, const float* d_cell_pos_f,
                                     double f32_eps, const int32_t* h_dims, int32_t shell, double near_rsq,
                                     const double* d_near_rsq, double rsq_max, int32_t cap,
                                     int32_t* d_nbr, int64_t ld_nbr, int32_t* d_nnear, int32_t* d_nnbr,
                                     const int32_t* d_order, int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!h_dims || !d_cell_pos || cap < 0 || ld_nbr < n_local || shell < 1 || !(near_rsq <= rsq_max) ||
      (d_cell_pos_f && !(f32_eps > 0.0)))
    return TMD_ERR_ARG;
  Tiers T{};
  T.r2[0] = near_rsq;
  T.nt = 1;
  T.d_r2 = d_near_rsq;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims, shell);
  C.order = d_order;
  C.cpf = d_cell_pos_f;
  C.f32_eps = f32_eps;
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

extern "C" int tmd_split_margin(const double* d_dispmax2, int32_t i0, int32_t i1, double floor_margin, double factor,
                                double cap, double cutoff, double* d_out, void* stream) {
  if (!d_dispmax2 || !d_out || i0 < 0 || i1 <= i0) return TMD_ERR_ARG;
  k_split_margin<<<1, 1, 0, as_stream(stream)>>>(d_dispmax2, i0, i1, floor_margin, factor, cap, cutoff, d_out);
  TMD_LAUNCH_CHECK("split_margin");
  return TMD_OK;
}
