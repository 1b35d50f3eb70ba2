// K8/K9 — halo-protocol building blocks (reference: comm.py:340-498).
//
// The host drives the three phases round by round (x, y, z) exactly as the
// reference's six-stencil pattern does; these kernels are the per-round data
// movement: order-preserving selection (flag + scan + scatter), gather with
// periodic shift into a send buffer or straight into this rank's ghost slots,
// in-place wrap for self-peer dimensions, the ownership check, and the
// flattened single-kernel ghost refresh used when every ghost is a periodic
// self-image (P = 1, and every self-peer dimension).
#include "tmd_common.cuh"

namespace tmd {

__global__ void k_flags(const double* __restrict__ x, int32_t n, int kind, double thr, double thr2,
                        int32_t* __restrict__ flag) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = x[i];
  bool f = kind == TMD_SEL_GE   ? (v >= thr)
           : kind == TMD_SEL_LT ? (v < thr)
           : kind == TMD_SEL_GT ? (v > thr)
                                : (v >= thr && v < thr2);
  flag[i] = f ? 1 : 0;
}

__global__ void k_compact(const int32_t* __restrict__ flag, const int32_t* __restrict__ off,
                          int32_t n, int32_t* __restrict__ idx, int32_t* __restrict__ count) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) idx[off[i]] = i;
  if (i == 0) *count = off[n];
}

__global__ void k_gather_shift(const double* __restrict__ pos, int64_t ld, const int32_t* __restrict__ idx,
                               int32_t k, double s0, double s1, double s2, int dim,
                               const double* __restrict__ sh, double* __restrict__ out, int64_t ld_out) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const int32_t j = idx[t];
  double s[3] = {s0, s1, s2};
  if (sh) s[dim] = sh[t];
#pragma unroll
  for (int q = 0; q < 3; ++q) out[q * ld_out + t] = add_rn(pos[q * ld + j], s[q]);
}

__global__ void k_plan_shift(const double* __restrict__ pos, int64_t ld, const int32_t* __restrict__ idx,
                             int32_t k, int dim, double s, double* __restrict__ sh) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const double x = pos[dim * ld + idx[t]];
  sh[t] = sub_rn(add_rn(x, s), x);
}

__global__ void k_wrap_self(double* __restrict__ pos, int64_t ld, int32_t n, int dim, double hi,
                            double lo, double sp, double sm) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = pos[dim * ld + i];
  // both entries test the round-start snapshot (comm.py:351, 356)
  if (x >= hi)
    pos[dim * ld + i] = add_rn(x, sp);
  else if (x < lo)
    pos[dim * ld + i] = add_rn(x, sm);
}

__global__ void k_check_owned(const double* __restrict__ pos, int64_t ld, int32_t n, double l0,
                              double l1, double l2, double h0, double h1, double h2, int64_t* st) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = pos[i], y = pos[ld + i], z = pos[2 * ld + i];
  bool in = (x >= l0 && x < h0) && (y >= l1 && y < h1) && (z >= l2 && z < h2);
  if (!in) raise_status(st, TMD_PROTOCOL, (unsigned long long)i);
}

__global__ void k_sync_flat(double* __restrict__ pos, int64_t ld, int32_t g0, int32_t k,
                            const int32_t* __restrict__ src, const double* __restrict__ sh) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const int32_t j = src[t];
#pragma unroll
  for (int q = 0; q < 3; ++q) pos[q * ld + g0 + t] = add_rn(pos[q * ld + j], sh[(int64_t)q * k + t]);
}

// ghosts [g0, g0 + kr) of one round, built from idx (locals or earlier ghosts)
__global__ void k_flatten_round(int32_t n_local, int32_t g0, int32_t kr, const int32_t* __restrict__ idx,
                                int dim, const double* __restrict__ sh, int32_t* __restrict__ src,
                                double* __restrict__ fsh, int64_t k_total) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kr) return;
  const int32_t p = idx[t];
  const int64_t me = (int64_t)(g0 - n_local) + t;  // index into the flat plan
  double s[3] = {0.0, 0.0, 0.0};
  int32_t root = p;
  if (p >= n_local) {  // parent is an earlier ghost: inherit its root and shifts
    const int64_t pp = (int64_t)(p - n_local);
    root = src[pp];
#pragma unroll
    for (int q = 0; q < 3; ++q) s[q] = fsh[q * k_total + pp];
  }
  s[dim] = sh[t];
  src[me] = root;
#pragma unroll
  for (int q = 0; q < 3; ++q) fsh[q * k_total + me] = s[q];
}

// both entries of a stencil round in one pass: flags for (+) and (-)
__global__ void k_flags_pair(const double* __restrict__ x, int32_t n, int ka, double ta, int kb, double tb,
                             int32_t* __restrict__ fa, int32_t* __restrict__ fb) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = x[i];
  auto pred = [v](int kind, double t) {
    return kind == TMD_SEL_GE ? (v >= t) : kind == TMD_SEL_LT ? (v < t) : (v > t);
  };
  fa[i] = pred(ka, ta) ? 1 : 0;
  fb[i] = pred(kb, tb) ? 1 : 0;
}

__global__ void k_compact_pair(const int32_t* __restrict__ fa, const int32_t* __restrict__ oa,
                               const int32_t* __restrict__ fb, const int32_t* __restrict__ ob, int32_t n,
                               int32_t* __restrict__ ia, int32_t* __restrict__ ib, int32_t* __restrict__ counts) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    if (fa[i]) ia[oa[i]] = i;
    if (fb[i]) ib[ob[i]] = i;
  }
  if (i == 0) {
    counts[0] = oa[n];
    counts[1] = ob[n];
  }
}

// ghosts g0 + t = pos[idx[t]] + S (comm.py:448-451), v = 0 (particles.py:148), and the
// plan's recorded shift along dim: sh[t] = (x + S_d) - x (comm.py:449)
__global__ void k_emit_ghosts(double* __restrict__ pos, double* __restrict__ vel, int64_t ld,
                              const int32_t* __restrict__ idx, int32_t k, double s0, double s1, double s2,
                              int dim, int32_t g0, double* __restrict__ sh) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const int32_t j = idx[t];
  const double s[3] = {s0, s1, s2};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double x = pos[q * ld + j];
    const double e = add_rn(x, s[q]);
    pos[q * ld + g0 + t] = e;
    vel[q * ld + g0 + t] = 0.0;
    if (q == dim) sh[t] = sub_rn(e, x);
  }
}

// Provenance of border copies: the owning rank, the owner's local index and
// the shift accumulated along each dimension.  A copy of a local p is
// (me, p, sh on dim); a copy of an earlier ghost inherits that ghost's
// provenance and adds this hop's recorded shift on `dim` (each dimension is
// crossed at most once, so x_root + s reproduces the hop-by-hop sum).
// Outputs go either to the ghost provenance arrays (self entries) or to an
// outgoing packet (remote entries).
__global__ void k_provenance(int32_t n_local, int32_t me, int32_t k, const int32_t* __restrict__ idx, int dim,
                             const double* __restrict__ sh, const int32_t* __restrict__ p_rank,
                             const int32_t* __restrict__ p_root, const double* __restrict__ p_sh, int64_t ld_p,
                             int32_t* __restrict__ o_rank, int32_t* __restrict__ o_root, double* __restrict__ o_sh,
                             int64_t ld_o) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const int32_t p = idx[t];
  double s[3] = {0.0, 0.0, 0.0};
  int32_t rank = me, root = p;
  if (p >= n_local) {
    const int64_t pp = (int64_t)(p - n_local);
    rank = p_rank[pp];
    root = p_root[pp];
#pragma unroll
    for (int q = 0; q < 3; ++q) s[q] = p_sh[q * ld_p + pp];
  }
  s[dim] = sh[t];
  o_rank[t] = rank;
  o_root[t] = root;
#pragma unroll
  for (int q = 0; q < 3; ++q) o_sh[q * ld_o + t] = s[q];
}

// Periodic borders in one pass when every stencil entry is self (P = 1).
// Round d of define_borders copies [0, n0) atoms with x_d > hi_d - r (shift
// -L_d) and x_d < lo_d + r (shift +L_d); earlier rounds only moved other
// coordinates, so atom i's copies are the product over d of {0} plus the
// options i's own x_d selects -- minus the identity.  Same set and same
// coordinates as the three rounds; the order is by local, then combination.
struct BorderBox {
  double thr_hi[3], thr_lo[3], s_hi[3], s_lo[3];
};

__device__ __forceinline__ int border_options(const BorderBox& B, int d, double x, double* opt) {
  int k = 0;
  opt[k++] = 0.0;
  if (x > B.thr_hi[d]) opt[k++] = B.s_hi[d];
  if (x < B.thr_lo[d]) opt[k++] = B.s_lo[d];
  return k;
}

__global__ void k_border_count(const double* __restrict__ pos, int64_t ld, int32_t n, BorderBox B,
                               int32_t* __restrict__ cnt) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int m = 1;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x = pos[d * ld + i];
    m *= 1 + (x > B.thr_hi[d]) + (x < B.thr_lo[d]);
  }
  cnt[i] = m - 1;
}

// Rank-grid position of this rank (dest of a copy = coords + per-dim offset).
struct RankGrid {
  int c[3], g[3];
  __device__ __forceinline__ int32_t index(int ox, int oy, int oz) const {
    const int x = (c[0] + ox + g[0]) % g[0], y = (c[1] + oy + g[1]) % g[1], z = (c[2] + oz + g[2]) % g[2];
    return (z * g[1] + y) * g[0] + x;  // comm.py rank_grid_index
  }
};

// Copies of local i at off[i] .. off[i+1]: coordinates to out_pos (3, ld_out)
// (+ v = 0 to out_vel when given), provenance root / recorded shift, and the
// destination rank (when d_dest is given; option +1 = the + neighbour).
__global__ void k_border_fill(const double* __restrict__ pos, int64_t ld, int32_t n, BorderBox B, RankGrid R,
                              const int32_t* __restrict__ off, double* __restrict__ out_pos, int64_t ld_out,
                              double* __restrict__ out_vel, int32_t* __restrict__ root, double* __restrict__ sh,
                              int64_t ld_sh, int32_t* __restrict__ dest, int64_t max_out) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t o = off[i];
  // copies past max_out are dropped (the caller compares off[n] with its room)
  if (off[i + 1] == o || (int64_t)o >= max_out) return;
  const double x[3] = {pos[i], pos[ld + i], pos[2 * ld + i]};
  double opt[3][3];
  int dir[3][3];
  int k[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int m = 0;
    opt[d][m] = 0.0;
    dir[d][m++] = 0;
    if (x[d] > B.thr_hi[d]) {
      opt[d][m] = B.s_hi[d];
      dir[d][m++] = 1;
    }
    if (x[d] < B.thr_lo[d]) {
      opt[d][m] = B.s_lo[d];
      dir[d][m++] = -1;
    }
    k[d] = m;
  }
  int32_t t = 0;
  for (int a = 0; a < k[0]; ++a)
    for (int b = 0; b < k[1]; ++b)
      for (int c = 0; c < k[2]; ++c) {
        if (a == 0 && b == 0 && c == 0) continue;
        const int64_t g = (int64_t)o + t++;
        if (g >= max_out) continue;
        const int sel[3] = {a, b, c};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double e = x[d], r = 0.0;
          if (sel[d]) {
            e = add_rn(x[d], opt[d][sel[d]]);
            r = sub_rn(e, x[d]);  // the recorded shift (comm.py:449)
          }
          out_pos[d * ld_out + g] = e;
          if (out_vel) out_vel[d * ld_out + g] = 0.0;
          sh[d * ld_sh + g] = r;
        }
        root[g] = i;
        if (dest) dest[g] = R.index(dir[0][a], dir[1][b], dir[2][c]);
      }
}

// Direct exchange (production path): self dimensions wrap in place
// (comm.py:351-356); for a remote dimension x_d >= hi_d goes to the + neighbour
// (shift -L_d at the global edge), x_d < lo_d to the - neighbour (+L_d).  The
// shift is applied in place; dest[i] = destination rank or -1 (stays).
struct Slab {
  double lo[3], hi[3], s_hi[3], s_lo[3];
};

__global__ void k_exchange_classify(double* __restrict__ pos, int64_t ld, int32_t n, Slab S, RankGrid R,
                                    int32_t* __restrict__ keep, int32_t* __restrict__ leave,
                                    int32_t* __restrict__ dest) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o[3] = {0, 0, 0};
  bool moved = false;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double x = pos[d * ld + i];
    if (x >= S.hi[d]) {
      pos[d * ld + i] = add_rn(x, S.s_hi[d]);
      if (R.g[d] > 1) {
        o[d] = 1;
        moved = true;
      }
    } else if (x < S.lo[d]) {
      pos[d * ld + i] = add_rn(x, S.s_lo[d]);
      if (R.g[d] > 1) {
        o[d] = -1;
        moved = true;
      }
    }
  }
  dest[i] = moved ? R.index(o[0], o[1], o[2]) : -1;
  keep[i] = moved ? 0 : 1;
  leave[i] = moved ? 1 : 0;
}

// Export table: ghost copies grouped by the local atom they mirror (counting
// sort by root index; order inside an atom is irrelevant).  Roots outside
// [0, n_local) are a protocol error.
__global__ void k_export_count(const int32_t* __restrict__ root, int32_t n_ex, int32_t n_local,
                               int32_t* __restrict__ cnt, int64_t* __restrict__ status,
                               const int32_t* __restrict__ d_n_ex) {
  int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (d_n_ex) n_ex = *d_n_ex;  // device-side count (grid sized for the maximum)
  if (e >= n_ex) return;
  const int32_t r = root[e];
  if (r < 0 || r >= n_local) {
    if (status) raise_status(status, TMD_PROTOCOL, (unsigned long long)e);
    return;
  }
  atomicAdd(&cnt[r], 1);
}

__global__ void k_export_scatter(const int32_t* __restrict__ root, const int32_t* __restrict__ rank,
                                 const int32_t* __restrict__ slot, const double* __restrict__ sh, int32_t n_ex,
                                 int32_t n_local, int64_t ld_sh, const int32_t* __restrict__ start, int32_t* __restrict__ fill,
                                 int32_t* __restrict__ o_rank, int32_t* __restrict__ o_slot,
                                 double* __restrict__ o_sh, int64_t ld_o, const int32_t* __restrict__ d_n_ex) {
  int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (d_n_ex) n_ex = *d_n_ex;
  if (e >= n_ex) return;
  const int32_t r = root[e];
  if (r < 0 || r >= n_local) return;
  const int32_t k = start[r] + atomicAdd(&fill[r], 1);
  o_rank[k] = rank[e];
  o_slot[k] = slot[e];
#pragma unroll
  for (int q = 0; q < 3; ++q) o_sh[q * ld_o + k] = sh[q * ld_sh + e];
}

}  // namespace tmd

using namespace tmd;

extern "C" int tmd_exports_build(int32_t n_local, int32_t n_ex, const int32_t* d_root, const int32_t* d_rank,
                                 const int32_t* d_slot, const double* d_sh, int64_t ld_sh, int32_t* d_start,
                                 int32_t* d_o_rank, int32_t* d_o_slot, double* d_o_sh, int64_t* d_status,
                                 void* stream) {
  return tmd_exports_build_dev(n_local, n_ex, nullptr, d_root, d_rank, d_slot, d_sh, ld_sh, d_start, d_o_rank,
                               d_o_slot, d_o_sh, n_ex, d_status, stream);
}

extern "C" int tmd_exports_build_dev(int32_t n_local, int32_t n_ex_max, const int32_t* d_n_ex, const int32_t* d_root,
                                     const int32_t* d_rank, const int32_t* d_slot, const double* d_sh, int64_t ld_sh,
                                     int32_t* d_start, int32_t* d_o_rank, int32_t* d_o_slot, double* d_o_sh,
                                     int64_t ld_o, int64_t* d_status, void* stream) {
  if (n_local < 0 || n_ex_max < 0 || ld_o < n_ex_max) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  keep_pool_memory();
  int32_t* cnt = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(&cnt, sizeof(int32_t) * (size_t)(2 * (int64_t)n_local + 2), s), "exports alloc");
  int32_t* fill = cnt + n_local + 1;
  TMD_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)(2 * (int64_t)n_local + 2), s), "exports memset");
  if (n_ex_max > 0) {
    k_export_count<<<grid_for(n_ex_max, 256), 256, 0, s>>>(d_root, n_ex_max, n_local, cnt, d_status, d_n_ex);
    TMD_LAUNCH_CHECK("exports count");
  }
  int rc = scan_exclusive(cnt, d_start, n_local, s);
  if (rc != TMD_OK) return rc;
  if (n_ex_max > 0) {
    k_export_scatter<<<grid_for(n_ex_max, 256), 256, 0, s>>>(d_root, d_rank, d_slot, d_sh, n_ex_max, n_local, ld_sh,
                                                             d_start, fill, d_o_rank, d_o_slot, d_o_sh, ld_o, d_n_ex);
    TMD_LAUNCH_CHECK("exports scatter");
  }
  TMD_CUDA_TRY(cudaFreeAsync(cnt, s), "exports free");
  return TMD_OK;
}

static BorderBox border_box(const double* h_thr_hi, const double* h_thr_lo, const double* h_s_hi,
                            const double* h_s_lo) {
  BorderBox B;
  for (int d = 0; d < 3; ++d) {
    B.thr_hi[d] = h_thr_hi[d];
    B.thr_lo[d] = h_thr_lo[d];
    B.s_hi[d] = h_s_hi[d];
    B.s_lo[d] = h_s_lo[d];
  }
  return B;
}

extern "C" int tmd_borders_count(const double* d_pos, int64_t ld, int32_t n_local, const double* h_thr_hi,
                                 const double* h_thr_lo, int32_t* d_off, void* stream) {
  if (!h_thr_hi || !h_thr_lo || !d_off || n_local < 0) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  keep_pool_memory();
  const double zero[3] = {0.0, 0.0, 0.0};
  BorderBox B = border_box(h_thr_hi, h_thr_lo, zero, zero);
  int32_t* cnt = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(&cnt, sizeof(int32_t) * (size_t)(n_local + 1), s), "borders alloc");
  if (n_local > 0) {
    k_border_count<<<grid_for(n_local, 256), 256, 0, s>>>(d_pos, ld, n_local, B, cnt);
    TMD_LAUNCH_CHECK("borders_count");
  }
  int rc = scan_exclusive(cnt, d_off, n_local, s);
  TMD_CUDA_TRY(cudaFreeAsync(cnt, s), "borders free");
  return rc;
}

static bool rank_grid(const int32_t* h_grid, RankGrid* R) {
  if (!h_grid) {
    *R = RankGrid{{0, 0, 0}, {1, 1, 1}};
    return true;
  }
  for (int d = 0; d < 3; ++d) {
    R->c[d] = h_grid[d];
    R->g[d] = h_grid[3 + d];
    if (R->g[d] < 1 || R->c[d] < 0 || R->c[d] >= R->g[d]) return false;
  }
  return true;
}

extern "C" int tmd_borders_fill(const double* d_pos, int64_t ld, int32_t n_local, const double* h_thr_hi,
                                const double* h_thr_lo, const double* h_s_hi, const double* h_s_lo,
                                const int32_t* h_grid, const int32_t* d_off, double* d_out_pos, int64_t ld_out,
                                double* d_out_vel, int32_t* d_root, double* d_sh, int64_t ld_sh, int32_t* d_dest,
                                void* stream) {
  return tmd_borders_fill_capped(d_pos, ld, n_local, h_thr_hi, h_thr_lo, h_s_hi, h_s_lo, h_grid, d_off, d_out_pos,
                                 ld_out, d_out_vel, d_root, d_sh, ld_sh, d_dest, INT64_MAX, stream);
}

extern "C" int tmd_borders_fill_capped(const double* d_pos, int64_t ld, int32_t n_local, const double* h_thr_hi,
                                       const double* h_thr_lo, const double* h_s_hi, const double* h_s_lo,
                                       const int32_t* h_grid, const int32_t* d_off, double* d_out_pos,
                                       int64_t ld_out, double* d_out_vel, int32_t* d_root, double* d_sh,
                                       int64_t ld_sh, int32_t* d_dest, int64_t max_out, void* stream) {
  if (!h_thr_hi || !h_thr_lo || !h_s_hi || !h_s_lo || !d_off || !d_out_pos) return TMD_ERR_ARG;
  RankGrid R;
  if (!rank_grid(h_grid, &R)) return TMD_ERR_ARG;
  if (n_local <= 0) return TMD_OK;
  BorderBox B = border_box(h_thr_hi, h_thr_lo, h_s_hi, h_s_lo);
  k_border_fill<<<grid_for(n_local, 128), 128, 0, as_stream(stream)>>>(d_pos, ld, n_local, B, R, d_off, d_out_pos,
                                                                      ld_out, d_out_vel, d_root, d_sh, ld_sh, d_dest,
                                                                      max_out);
  TMD_LAUNCH_CHECK("borders_fill");
  return TMD_OK;
}

extern "C" int tmd_exchange_classify(double* d_pos, int64_t ld, int32_t n, const double* h_lo, const double* h_hi,
                                     const double* h_s_hi, const double* h_s_lo, const int32_t* h_grid,
                                     int32_t* d_dest, int32_t* d_keep_idx, int32_t* d_leave_idx,
                                     int32_t* d_counts, int32_t* d_scratch, void* stream) {
  if (!h_lo || !h_hi || !h_s_hi || !h_s_lo || !h_grid) return TMD_ERR_ARG;
  RankGrid R;
  if (!rank_grid(h_grid, &R)) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  if (n <= 0) {
    TMD_CUDA_TRY(cudaMemsetAsync(d_counts, 0, 2 * sizeof(int32_t), s), "exchange_classify");
    return TMD_OK;
  }
  Slab S;
  for (int d = 0; d < 3; ++d) {
    S.lo[d] = h_lo[d];
    S.hi[d] = h_hi[d];
    S.s_hi[d] = h_s_hi[d];
    S.s_lo[d] = h_s_lo[d];
  }
  int32_t* buf = d_scratch;
  if (!buf) {
    keep_pool_memory();
    TMD_CUDA_TRY(cudaMallocAsync(&buf, sizeof(int32_t) * (size_t)(4 * (int64_t)n + 2), s), "exchange alloc");
  }
  int32_t *fa = buf, *fb = buf + n, *oa = buf + 2 * (int64_t)n, *ob = oa + n + 1;
  k_exchange_classify<<<grid_for(n, 256), 256, 0, s>>>(d_pos, ld, n, S, R, fa, fb, d_dest);
  TMD_LAUNCH_CHECK("exchange_classify");
  int rc = scan_exclusive(fa, oa, n, s);
  if (rc == TMD_OK) rc = scan_exclusive(fb, ob, n, s);
  if (rc != TMD_OK) return rc;
  k_compact_pair<<<grid_for(n, 256), 256, 0, s>>>(fa, oa, fb, ob, n, d_keep_idx, d_leave_idx, d_counts);
  TMD_LAUNCH_CHECK("exchange compact");
  if (!d_scratch) TMD_CUDA_TRY(cudaFreeAsync(buf, s), "exchange free");
  return TMD_OK;
}

extern "C" int tmd_ghost_provenance(int32_t n_local, int32_t me, int32_t k, const int32_t* d_idx, int32_t dim,
                                    const double* d_sh, const int32_t* d_p_rank, const int32_t* d_p_root,
                                    const double* d_p_sh, int64_t ld_p, int32_t* d_o_rank, int32_t* d_o_root,
                                    double* d_o_sh, int64_t ld_o, void* stream) {
  if (k <= 0) return TMD_OK;
  if (dim < 0 || dim > 2) return TMD_ERR_ARG;
  k_provenance<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(n_local, me, k, d_idx, dim, d_sh, d_p_rank, d_p_root,
                                                                d_p_sh, ld_p, d_o_rank, d_o_root, d_o_sh, ld_o);
  TMD_LAUNCH_CHECK("ghost_provenance");
  return TMD_OK;
}

extern "C" int tmd_select_pair(const double* d_coord, int32_t n, int32_t kind_a, double thr_a, int32_t kind_b,
                               double thr_b, int32_t* d_idx_a, int32_t* d_idx_b, int32_t* d_counts,
                               void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) {
    TMD_CUDA_TRY(cudaMemsetAsync(d_counts, 0, 2 * sizeof(int32_t), s), "select_pair");
    return TMD_OK;
  }
  keep_pool_memory();
  int32_t* buf = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(&buf, sizeof(int32_t) * (size_t)(4 * (int64_t)n + 2), s), "select_pair alloc");
  int32_t *fa = buf, *fb = buf + n, *oa = buf + 2 * (int64_t)n, *ob = oa + n + 1;
  k_flags_pair<<<grid_for(n, 256), 256, 0, s>>>(d_coord, n, kind_a, thr_a, kind_b, thr_b, fa, fb);
  TMD_LAUNCH_CHECK("select_pair flags");
  int rc = scan_exclusive(fa, oa, n, s);
  if (rc == TMD_OK) rc = scan_exclusive(fb, ob, n, s);
  if (rc != TMD_OK) return rc;
  k_compact_pair<<<grid_for(n, 256), 256, 0, s>>>(fa, oa, fb, ob, n, d_idx_a, d_idx_b, d_counts);
  TMD_LAUNCH_CHECK("select_pair compact");
  TMD_CUDA_TRY(cudaFreeAsync(buf, s), "select_pair free");
  return TMD_OK;
}

extern "C" int tmd_emit_ghosts(double* d_pos, double* d_vel, int64_t ld, const int32_t* d_idx, int32_t k,
                               const double* h_shift, int32_t dim, int32_t g0, double* d_sh, void* stream) {
  if (k <= 0) return TMD_OK;
  k_emit_ghosts<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(d_pos, d_vel, ld, d_idx, k, h_shift[0],
                                                                 h_shift[1], h_shift[2], dim, g0, d_sh);
  TMD_LAUNCH_CHECK("emit_ghosts");
  return TMD_OK;
}

extern "C" int tmd_select(const double* d_coord, int32_t n, int32_t kind, double thr, double thr2,
                          int32_t* d_idx, int32_t* d_count, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) {
    TMD_CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int32_t), s), "select");
    return TMD_OK;
  }
  keep_pool_memory();
  int32_t* flag = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(&flag, sizeof(int32_t) * (size_t)(2 * n + 1), s), "select alloc");
  int32_t* off = flag + n;
  k_flags<<<grid_for(n, 256), 256, 0, s>>>(d_coord, n, kind, thr, thr2, flag);
  TMD_LAUNCH_CHECK("select flags");
  int rc = scan_exclusive(flag, off, n, s);
  if (rc != TMD_OK) return rc;
  k_compact<<<grid_for(n, 256), 256, 0, s>>>(flag, off, n, d_idx, d_count);
  TMD_LAUNCH_CHECK("select compact");
  TMD_CUDA_TRY(cudaFreeAsync(flag, s), "select free");
  return TMD_OK;
}

extern "C" int tmd_gather_shift(const double* d_pos, int64_t ld, const int32_t* d_idx, int32_t k,
                                const double* h_shift, int32_t dim, const double* d_shift_d,
                                double* d_out, int64_t ld_out, void* stream) {
  if (k <= 0) return TMD_OK;
  double s0 = h_shift ? h_shift[0] : 0.0, s1 = h_shift ? h_shift[1] : 0.0,
         s2 = h_shift ? h_shift[2] : 0.0;
  k_gather_shift<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(d_pos, ld, d_idx, k, s0, s1, s2,
                                                                  dim, d_shift_d, d_out, ld_out);
  TMD_LAUNCH_CHECK("gather_shift");
  return TMD_OK;
}

extern "C" int tmd_plan_shift(const double* d_pos, int64_t ld, const int32_t* d_idx, int32_t k,
                              int32_t dim, double s, double* d_sh, void* stream) {
  if (k <= 0) return TMD_OK;
  k_plan_shift<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(d_pos, ld, d_idx, k, dim, s, d_sh);
  TMD_LAUNCH_CHECK("plan_shift");
  return TMD_OK;
}

extern "C" int tmd_wrap_self(double* d_pos, int64_t ld, int32_t n, int32_t dim, double hi, double lo,
                             double s_plus, double s_minus, void* stream) {
  if (n <= 0) return TMD_OK;
  k_wrap_self<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d_pos, ld, n, dim, hi, lo, s_plus,
                                                               s_minus);
  TMD_LAUNCH_CHECK("wrap_self");
  return TMD_OK;
}

extern "C" int tmd_check_owned(const double* d_pos, int64_t ld, int32_t n, const double* h_lo,
                               const double* h_hi, int64_t* d_status, void* stream) {
  if (n <= 0) return TMD_OK;
  k_check_owned<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(
      d_pos, ld, n, h_lo[0], h_lo[1], h_lo[2], h_hi[0], h_hi[1], h_hi[2], d_status);
  TMD_LAUNCH_CHECK("check_owned");
  return TMD_OK;
}

extern "C" int tmd_sync_flat(double* d_pos, int64_t ld, int32_t g0, int32_t k, const int32_t* d_src,
                             const double* d_sh, void* stream) {
  if (k <= 0) return TMD_OK;
  k_sync_flat<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(d_pos, ld, g0, k, d_src, d_sh);
  TMD_LAUNCH_CHECK("sync_flat");
  return TMD_OK;
}

extern "C" int tmd_flatten_round(int32_t n_local, int32_t g0, int32_t k, const int32_t* d_idx,
                                 int32_t dim, const double* d_sh, int32_t* d_src, double* d_flat_sh,
                                 int64_t k_total, void* stream) {
  if (k <= 0) return TMD_OK;
  k_flatten_round<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(n_local, g0, k, d_idx, dim, d_sh,
                                                                   d_src, d_flat_sh, k_total);
  TMD_LAUNCH_CHECK("flatten_round");
  return TMD_OK;
}

// ---------------------------------------------------------------------------
// Direct-protocol bookkeeping on the device (exchange / borders at P > 1):
// grouping of records by destination rank, packing of (x, v) rows for the
// all-to-all, appending received rows to the store, and the slots of border
// copies on their receivers.  Replaces host-side sorts and index arithmetic.
// ---------------------------------------------------------------------------
namespace tmd {

constexpr int kGroupThreads = 1024;
constexpr int kGroupWarps = kGroupThreads / 32;
constexpr int kGroupMaxRanks = 8;

// Stable counting sort of m records by rank rk[t] in [0, P), in three passes
// over blocks of kGroupChunk records: per-block rank counts, per-block first
// slots (one warp), and the stable scatter (each warp ballots every rank).
constexpr int kGroupChunk = kGroupThreads * 4;  // records per block

// pass 1: per-block, per-rank record counts (warp-aggregated shared atomics)
__global__ void __launch_bounds__(kGroupThreads) k_group_count(const int32_t* __restrict__ rk, int32_t m, int P,
                                                               int32_t* __restrict__ block_counts) {
  __shared__ int32_t s_cnt[kGroupMaxRanks];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < kGroupMaxRanks) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int32_t lo = blockIdx.x * kGroupChunk, hi = min(m, lo + kGroupChunk);
  for (int32_t t = lo + threadIdx.x; t < lo + kGroupChunk; t += blockDim.x) {
    const int r = t < hi ? rk[t] : -1;
    for (int q = 0; q < P; ++q) {
      const unsigned b = __ballot_sync(0xffffffffu, r == q);
      if (lane == 0 && b) atomicAdd(&s_cnt[q], __popc(b));
    }
  }
  __syncthreads();
  if (threadIdx.x < P) block_counts[blockIdx.x * kGroupMaxRanks + threadIdx.x] = s_cnt[threadIdx.x];
}

// pass 2: group sizes, and each block's first output slot per rank (in place)
__global__ void k_group_offsets(int32_t* __restrict__ block_counts, int nb, int P, int32_t* __restrict__ counts) {
  __shared__ int32_t s_tot[kGroupMaxRanks];
  const int q = threadIdx.x;
  if (q < P) {
    int32_t acc = 0;
    for (int b = 0; b < nb; ++b) {
      const int32_t c = block_counts[b * kGroupMaxRanks + q];
      block_counts[b * kGroupMaxRanks + q] = acc;
      acc += c;
    }
    s_tot[q] = acc;
    counts[q] = acc;
  }
  __syncthreads();
  if (q < P) {
    int32_t start = 0;
    for (int r = 0; r < q; ++r) start += s_tot[r];
    for (int b = 0; b < nb; ++b) block_counts[b * kGroupMaxRanks + q] += start;
  }
}

// pass 3: stable scatter.  A record's position is (its block's first slot for
// its rank) + (its rank's records in earlier rounds and warps of the block) +
// (its rank's lanes below it).  out_ids[pos] = ids[t] (t itself when ids is
// null), out_rank[pos] = rank.
__global__ void __launch_bounds__(kGroupThreads) k_group_scatter(const int32_t* __restrict__ rk,
                                                                 const int32_t* __restrict__ ids, int32_t m, int P,
                                                                 const int32_t* __restrict__ block_first,
                                                                 int32_t* __restrict__ out_ids,
                                                                 int32_t* __restrict__ out_rank) {
  __shared__ int32_t s_run[kGroupMaxRanks];
  __shared__ int32_t s_warp[kGroupMaxRanks][kGroupWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x < P) s_run[threadIdx.x] = block_first[blockIdx.x * kGroupMaxRanks + threadIdx.x];
  __syncthreads();
  const int32_t lo = blockIdx.x * kGroupChunk, hi = min(m, lo + kGroupChunk);
  for (int32_t base = lo; base < hi; base += blockDim.x) {
    const int32_t t = base + threadIdx.x;
    int r = t < hi ? rk[t] : -1;
    if (r >= P) r = -1;  // records outside [0, P) drop out
    unsigned mine = 0;
    for (int q = 0; q < P; ++q) {
      const unsigned b = __ballot_sync(0xffffffffu, r == q);
      if (r == q) mine = b;
      if (lane == 0) s_warp[q][wid] = __popc(b);
    }
    __syncthreads();
    if (r >= 0) {
      int32_t pos = s_run[r] + __popc(mine & lt);
      for (int w = 0; w < wid; ++w) pos += s_warp[r][w];
      out_ids[pos] = ids ? ids[t] : t;
      if (out_rank) out_rank[pos] = r;
    }
    __syncthreads();
    if (threadIdx.x < P) {
      int32_t c = 0;
      for (int w = 0; w < kGroupWarps; ++w) c += s_warp[threadIdx.x][w];
      s_run[threadIdx.x] += c;
    }
    __syncthreads();
  }
}

// rows[t] = (x, y, z[, vx, vy, vz]) of atom idx[t] (+ shift on x): the
// all-to-all payload, one contiguous row per record
__global__ void k_pack_rows(const double* __restrict__ pos, const double* __restrict__ vel, int64_t ld,
                            const int32_t* __restrict__ idx, int32_t k, int width, double* __restrict__ rows) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const int32_t j = idx[t];
  double* o = rows + (int64_t)t * width;
  o[0] = pos[j];
  o[1] = pos[ld + j];
  o[2] = pos[2 * ld + j];
  if (width == 6) {
    o[3] = vel[j];
    o[4] = vel[ld + j];
    o[5] = vel[2 * ld + j];
  }
}

// the inverse: rows (k, width) into the store at slots [at, at + k); width 3
// rows are ghosts (v = 0)
__global__ void k_unpack_rows(const double* __restrict__ rows, int32_t k, int width, double* __restrict__ pos,
                              double* __restrict__ vel, int64_t ld, int32_t at) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const double* r = rows + (int64_t)t * width;
  const int32_t s = at + t;
  pos[s] = r[0];
  pos[ld + s] = r[1];
  pos[2 * ld + s] = r[2];
  vel[s] = width == 6 ? r[3] : 0.0;
  vel[ld + s] = width == 6 ? r[4] : 0.0;
  vel[2 * ld + s] = width == 6 ? r[5] : 0.0;
}

// slot of the t-th grouped border copy on its receiver: base[rank] + t
struct RankBase {
  int64_t v[kGroupMaxRanks];
};
__global__ void k_border_slots(const int32_t* __restrict__ rank, int32_t m, RankBase b, int32_t* __restrict__ slot) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) slot[t] = (int32_t)(b.v[rank[t]] + t);
}

__global__ void k_gather_i32x(const int32_t* __restrict__ src, const int32_t* __restrict__ idx, int32_t n,
                              int32_t* __restrict__ out) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = src[idx[t]];
}

}  // namespace tmd

extern "C" int tmd_group_by_rank(const int32_t* d_rank, const int32_t* d_ids, int32_t m, int32_t n_ranks,
                                 int32_t* d_out_ids, int32_t* d_out_rank, int32_t* d_counts, void* stream) {
  if (n_ranks < 1 || n_ranks > kGroupMaxRanks || !d_counts || m < 0) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  if (m == 0) {
    TMD_CUDA_TRY(cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * n_ranks, s), "group_by_rank");
    return TMD_OK;
  }
  if (!d_rank || !d_out_ids) return TMD_ERR_ARG;
  // per-block counts live in this stream's reduction scratch (stream-ordered use)
  const int nb = (int)((m + kGroupChunk - 1) / kGroupChunk);
  ReduceScratch rs;
  const int rc = reduce_scratch(&rs, nb, kGroupMaxRanks, s);
  if (rc != TMD_OK) return rc;
  int32_t* blk = reinterpret_cast<int32_t*>(rs.partials);
  k_group_count<<<nb, kGroupThreads, 0, s>>>(d_rank, m, n_ranks, blk);
  TMD_LAUNCH_CHECK("group_by_rank");
  k_group_offsets<<<1, 32, 0, s>>>(blk, nb, n_ranks, d_counts);
  TMD_LAUNCH_CHECK("group_by_rank");
  k_group_scatter<<<nb, kGroupThreads, 0, s>>>(d_rank, d_ids, m, n_ranks, blk, d_out_ids, d_out_rank);
  TMD_LAUNCH_CHECK("group_by_rank");
  return TMD_OK;
}

extern "C" int tmd_pack_rows(const double* d_pos, const double* d_vel, int64_t ld, const int32_t* d_idx, int32_t k,
                             int32_t width, double* d_rows, void* stream) {
  if (k <= 0) return TMD_OK;
  if ((width != 3 && width != 6) || (width == 6 && !d_vel)) return TMD_ERR_ARG;
  k_pack_rows<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(d_pos, d_vel, ld, d_idx, k, width, d_rows);
  TMD_LAUNCH_CHECK("pack_rows");
  return TMD_OK;
}

extern "C" int tmd_unpack_rows(const double* d_rows, int32_t k, int32_t width, double* d_pos, double* d_vel,
                               int64_t ld, int32_t at, void* stream) {
  if (k <= 0) return TMD_OK;
  if (width != 3 && width != 6) return TMD_ERR_ARG;
  k_unpack_rows<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(d_rows, k, width, d_pos, d_vel, ld, at);
  TMD_LAUNCH_CHECK("unpack_rows");
  return TMD_OK;
}

extern "C" int tmd_border_slots(const int32_t* d_rank, int32_t m, int32_t n_ranks, const int64_t* h_base,
                                int32_t* d_slot, void* stream) {
  if (m <= 0) return TMD_OK;
  if (n_ranks < 1 || n_ranks > kGroupMaxRanks || !h_base) return TMD_ERR_ARG;
  RankBase b{};
  for (int q = 0; q < n_ranks; ++q) b.v[q] = h_base[q];
  k_border_slots<<<grid_for(m, 256), 256, 0, as_stream(stream)>>>(d_rank, m, b, d_slot);
  TMD_LAUNCH_CHECK("border_slots");
  return TMD_OK;
}

extern "C" int tmd_gather_i32(const int32_t* d_src, const int32_t* d_idx, int32_t n, int32_t* d_out, void* stream) {
  if (n <= 0) return TMD_OK;
  k_gather_i32x<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d_src, d_idx, n, d_out);
  TMD_LAUNCH_CHECK("gather_i32");
  return TMD_OK;
}
