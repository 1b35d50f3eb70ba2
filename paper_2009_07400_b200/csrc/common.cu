// Library-wide state: last error, device info, reduction scratch, int32 scan.
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "tmd_common.cuh"

namespace tmd {

static thread_local char g_err[512] = "";
static unsigned long long g_launches = 0;

void count_launch() { __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED); }

void set_last_error(const char* where, cudaError_t e) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorName(e),
                cudaGetErrorString(e));
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

// One reduction scratch per (device, stream), grown on demand (never shrinks):
// kernels on different streams -- ranks of an in-process run (loopback.py),
// or a caller's own streams -- never share partials or the last-block counter.
int reduce_scratch(ReduceScratch* rs, int blocks, int nv, cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, ReduceScratch> per_stream;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  ReduceScratch& r = per_stream[{dev, stream}];
  int need = blocks * (nv < 8 ? 8 : nv);
  if (r.partials == nullptr || r.max_blocks < need) {
    if (r.partials) {
      // only this stream's kernels use the old buffers
      cudaStreamSynchronize(stream);
      cudaFree(r.partials);
      cudaFree(r.counter);
      r.partials = nullptr;
    }
    // generous first size and doubling: a regrow synchronises the stream, and
    // atom counts drift with every migration
    int cap = need < (1 << 20) ? (1 << 20) : 2 * need;
    TMD_CUDA_TRY(cudaMalloc(&r.partials, sizeof(double) * (size_t)cap), "reduce_scratch");
    TMD_CUDA_TRY(cudaMalloc(&r.counter, sizeof(unsigned int) * 64), "reduce_scratch");
    TMD_CUDA_TRY(cudaMemsetAsync(r.counter, 0, sizeof(unsigned int) * 64, stream), "reduce_scratch");
    r.max_blocks = cap;
  }
  *rs = r;
  return TMD_OK;
}

// ---------------------------------------------------------------------------
// exclusive scan: 1024 threads x 4 items per block, recursive over block sums
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int32_t block_exclusive(int32_t v, int32_t* warp_tot, int32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int32_t w = warp_tot[lane];
    int32_t winc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t t = __shfl_up_sync(0xffffffffu, winc, o);
      if (lane >= o) winc += t;
    }
    warp_tot[lane] = winc - w;
    if (lane == 31) *total = winc;
  }
  __syncthreads();
  return warp_tot[wid] + inc - v;
}

// Scans in[0, n) padded with zeros to m = n + 1 outputs.
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const int32_t* __restrict__ in,
                                                              int32_t* __restrict__ out,
                                                              int32_t* __restrict__ tile_sums,
                                                              int64_t n, int64_t m) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t total;
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t v[kScanItems];
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    v[k] = (i < n) ? in[i] : 0;
    s += v[k];
  }
  int32_t run = block_exclusive(s, warp_tot, &total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    if (i < m) out[i] = run;
    run += v[k];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_add(int32_t* __restrict__ out, const int32_t* __restrict__ tile_off, int64_t m) {
  int64_t i = (int64_t)blockIdx.x * kScanTile + threadIdx.x;
  int32_t off = tile_off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k, i += kScanThreads)
    if (i < m) out[i] += off;
}

// Keep freed stream-ordered allocations in the device pool instead of
// returning them to the driver at every synchronisation (the default), so the
// per-epoch scratch of binning/selection costs no driver allocations.
void keep_pool_memory() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev & 63]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev & 63] = true;
}

int scan_exclusive(const int32_t* d_in, int32_t* d_out, int64_t n, cudaStream_t s) {
  int64_t m = n + 1;
  int64_t tiles = (m + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    k_scan_tiles<<<1, kScanThreads, 0, s>>>(d_in, d_out, nullptr, n, m);
    TMD_LAUNCH_CHECK("scan_exclusive");
    return TMD_OK;
  }
  int32_t* sums = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(&sums, sizeof(int32_t) * (size_t)(2 * tiles + 2), s), "scan alloc");
  int32_t* offs = sums + tiles;
  k_scan_tiles<<<(unsigned)tiles, kScanThreads, 0, s>>>(d_in, d_out, sums, n, m);
  TMD_LAUNCH_CHECK("scan_exclusive tiles");
  int rc = scan_exclusive(sums, offs, tiles, s);  // offs has tiles + 1 entries
  if (rc != TMD_OK) return rc;
  k_scan_add<<<(unsigned)tiles, kScanThreads, 0, s>>>(d_out, offs, m);
  TMD_LAUNCH_CHECK("scan_exclusive add");
  TMD_CUDA_TRY(cudaFreeAsync(sums, s), "scan free");
  return TMD_OK;
}

}  // namespace tmd

extern "C" {

int tmd_version(void) { return 1; }

int64_t tmd_launch_count(void) { return (int64_t)__atomic_load_n(&tmd::g_launches, __ATOMIC_RELAXED); }

const char* tmd_last_error(void) { return tmd::g_err; }

int tmd_device_info(int* sm, int* major, int* minor, int64_t* l2) {
  int dev = 0;
  TMD_CUDA_TRY(cudaGetDevice(&dev), "device_info");
  cudaDeviceProp p;
  TMD_CUDA_TRY(cudaGetDeviceProperties(&p, dev), "device_info");
  if (sm) *sm = p.multiProcessorCount;
  if (major) *major = p.major;
  if (minor) *minor = p.minor;
  if (l2) *l2 = p.l2CacheSize;
  return TMD_OK;
}

__global__ void k_status_reset(int64_t* st) {
  if (threadIdx.x == 0) {
    st[0] = 0;
    st[1] = (int64_t)-1;  // all ones: atomicMin identity (as unsigned)
    st[2] = 0;
    st[3] = 0;
  }
}

int tmd_status_reset(int64_t* d_status, void* stream) {
  k_status_reset<<<1, 32, 0, tmd::as_stream(stream)>>>(d_status);
  TMD_LAUNCH_CHECK("status_reset");
  return TMD_OK;
}

// [status code, d_vals[0 .. n)] as doubles in one buffer: the host reads an
// epoch's status and guard maxima with one copy
__global__ void k_check_pack(const int64_t* __restrict__ st, const double* __restrict__ vals, int32_t n,
                             double* __restrict__ out) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) out[0] = (double)st[0];
  if (t < n) out[1 + t] = vals[t];
}

// Allocate the stream's reduction scratch now (a device allocation orders all
// streams of the context: with in-process ranks whose barrier kernels wait for
// each other, it must not happen in the middle of a run).
int tmd_prepare_stream(void* stream) {
  tmd::ReduceScratch rs;
  return tmd::reduce_scratch(&rs, 1, 8, tmd::as_stream(stream));
}

int tmd_check_pack(const int64_t* d_status, const double* d_vals, int32_t n, double* d_out, void* stream) {
  if (!d_status || !d_out || n < 0 || (n > 0 && !d_vals)) return TMD_ERR_ARG;
  k_check_pack<<<tmd::grid_for(n > 0 ? n : 1, 256), 256, 0, tmd::as_stream(stream)>>>(d_status, d_vals, n, d_out);
  TMD_LAUNCH_CHECK("check_pack");
  return TMD_OK;
}

int tmd_copy_rows(const double* d_src, int64_t ld_src, double* d_dst, int64_t ld_dst, int32_t rows, int64_t count,
                  void* stream) {
  if (count <= 0) return TMD_OK;
  if (!d_src || !d_dst || rows < 1 || ld_src < count || ld_dst < count) return TMD_ERR_ARG;
  TMD_CUDA_TRY(cudaMemcpy2DAsync(d_dst, sizeof(double) * ld_dst, d_src, sizeof(double) * ld_src,
                                 sizeof(double) * count, rows, cudaMemcpyDeviceToDevice, tmd::as_stream(stream)),
               "copy_rows");
  return TMD_OK;
}

// ---- peer memory for the fused ghost refresh ------------------------------
// A pointer inside a cudaMalloc'd block (the caching allocator hands out
// sub-ranges) is exported as the block's IPC handle plus the byte offset.
typedef int (*AddressRangeFn)(unsigned long long* base, size_t* size, unsigned long long ptr);

int tmd_ipc_handle(const void* d_ptr, void* handle_out, int64_t* offset_out) {
  static AddressRangeFn range = nullptr;
  if (!range) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    TMD_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q), "ipc entry point");
    if (q != cudaDriverEntryPointSuccess || !fn) {
      tmd::set_last_error("ipc: cuMemGetAddressRange unavailable", cudaErrorNotSupported);
      return TMD_ERR_CUDA;
    }
    range = (AddressRangeFn)fn;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)d_ptr) != 0) {
    tmd::set_last_error("ipc: cuMemGetAddressRange", cudaErrorInvalidValue);
    return TMD_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  TMD_CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base), "ipc get handle");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((unsigned long long)d_ptr - base);
  return TMD_OK;
}

int tmd_ipc_open(const void* handle, int64_t offset, void** d_ptr_out, void** d_base_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  TMD_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
  *d_base_out = base;
  *d_ptr_out = (char*)base + offset;
  return TMD_OK;
}

int tmd_ipc_close(void* d_base) {
  TMD_CUDA_TRY(cudaIpcCloseMemHandle(d_base), "ipc close");
  return TMD_OK;
}

int tmd_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

}  // extern "C"
