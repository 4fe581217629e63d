// curve.cu — K1: token orderings on device (curve.cpp:39-185 restated for sm_100a).
//
// Every ordering is an order-preserving compaction of a "virtual" index space
// onto lattice cells: the enclosing 2^b cube walked by Skilling's transform
// (hilbert3d), per-frame 2^b squares (hilbert2d), padded 4^3 cubes (block3d).
// Cells outside the lattice are skipped, exactly like the reference's
// push_back loop (curve.cpp:105-110). Three launches: per-chunk valid counts,
// one-block exclusive scan of the chunk counts, then an in-chunk scan that
// writes forward[pos] = raster and (optionally) inverse[raster] = pos.
// Integer-only and negligible (~2M cells at HunyuanVideo); computed once per
// geometry and cached by the handle.
#include "common.cuh"

namespace dfsgpu {

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 16;
constexpr int kChunk = kThreads * kPerThread;

struct Geometry {
  int ordering;
  int64_t f, h, w;
  int bits;         // per-axis bits of the enclosing power of two (hilbert)
  int64_t virt;     // size of the virtual index space
  int64_t cf, ch, cw;  // cube grid (block3d)
};

// curve.cpp:50-81 (Skilling "transpose -> axes"), NDims = 2 or 3
template <int ND>
__device__ __forceinline__ void skilling(uint64_t index, int bits, uint32_t (&x)[ND]) {
#pragma unroll
  for (int a = 0; a < ND; ++a) x[a] = 0;
  if (bits == 0) return;
  for (int lvl = 0; lvl < bits; ++lvl) {
    const uint64_t group = index >> ((bits - 1 - lvl) * ND);
#pragma unroll
    for (int a = 0; a < ND; ++a) x[a] |= uint32_t((group >> (ND - 1 - a)) & 1u) << (bits - 1 - lvl);
  }
  const uint32_t t = x[ND - 1] >> 1;
#pragma unroll
  for (int a = ND - 1; a > 0; --a) x[a] ^= x[a - 1];
  x[0] ^= t;
  const uint32_t top = 1u << bits;
  for (uint32_t q = 2; q != top; q <<= 1) {
    const uint32_t p = q - 1;
#pragma unroll
    for (int a = ND - 1; a >= 0; --a) {
      if (x[a] & q) {
        x[0] ^= p;
      } else {
        const uint32_t s = (x[0] ^ x[a]) & p;
        x[0] ^= s;
        x[a] ^= s;
      }
    }
  }
}

// raster index of virtual cell v, or -1 when it lies outside the lattice
__device__ __forceinline__ int64_t virtual_cell(const Geometry& g, int64_t v) {
  switch (g.ordering) {
    case DFS_RASTER:
      return v;
    case DFS_HILBERT3D: {
      uint32_t a[3];
      skilling<3>(uint64_t(v), g.bits, a);
      if (a[0] < g.f && a[1] < g.h && a[2] < g.w) return (int64_t(a[0]) * g.h + a[1]) * g.w + a[2];
      return -1;
    }
    case DFS_HILBERT2D: {
      const int64_t cells = int64_t(1) << (2 * g.bits);
      const int64_t t = v / cells;
      uint32_t a[2];
      skilling<2>(uint64_t(v % cells), g.bits, a);
      if (a[0] < g.h && a[1] < g.w) return (t * g.h + a[0]) * g.w + a[1];
      return -1;
    }
    default: {  // DFS_BLOCK3D, curve.cpp:135-154
      const int64_t cube = v >> 6, local = v & 63;
      const int64_t cx = cube % g.cw, cy = (cube / g.cw) % g.ch, ct = cube / (g.cw * g.ch);
      const int64_t t = ct * 4 + (local >> 4), y = cy * 4 + ((local >> 2) & 3), x = cx * 4 + (local & 3);
      if (t < g.f && y < g.h && x < g.w) return (t * g.h + y) * g.w + x;
      return -1;
    }
  }
}

// exclusive block scan of one int per thread; returns the block total in *total
__device__ __forceinline__ int block_exclusive_scan(int v, int* total) {
  __shared__ int warp_tot[kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < kThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kThreads / 32) warp_tot[lane] = w;
  }
  __syncthreads();
  const int before = wid ? warp_tot[wid - 1] : 0;
  if (total) *total = warp_tot[kThreads / 32 - 1];
  const int excl = before + x - v;
  __syncthreads();
  return excl;
}

__global__ void __launch_bounds__(kThreads) count_kernel(Geometry g, int* chunk_counts) {
  const int64_t base = int64_t(blockIdx.x) * kChunk + int64_t(threadIdx.x) * kPerThread;
  int c = 0;
#pragma unroll 4
  for (int j = 0; j < kPerThread; ++j) {
    const int64_t v = base + j;
    if (v < g.virt && virtual_cell(g, v) >= 0) ++c;
  }
  int total;
  block_exclusive_scan(c, &total);
  if (threadIdx.x == 0) chunk_counts[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) scan_chunks_kernel(int* counts, int nchunks) {
  // single block, sequential over 1024-wide tiles with a running carry
  __shared__ int buf[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nchunks; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < nchunks ? counts[i] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int y = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < nchunks) counts[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) write_kernel(Geometry g, const int* chunk_offsets,
                                                         uint32_t* fwd, uint32_t* inv) {
  const int64_t base = int64_t(blockIdx.x) * kChunk + int64_t(threadIdx.x) * kPerThread;
  int64_t cell[kPerThread];
  int c = 0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    const int64_t v = base + j;
    cell[j] = v < g.virt ? virtual_cell(g, v) : -1;
    c += cell[j] >= 0;
  }
  int pos = chunk_offsets[blockIdx.x] + block_exclusive_scan(c, nullptr);
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    if (cell[j] < 0) continue;
    fwd[pos] = uint32_t(cell[j]);
    if (inv) inv[cell[j]] = uint32_t(pos);
    ++pos;
  }
}

__global__ void invert_kernel(const uint32_t* __restrict__ fwd, int64_t n, uint32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    if (int64_t(fwd[i]) < n) inv[fwd[i]] = uint32_t(i);  // out-of-range entries: no wild write
}

__global__ void histogram_kernel(const uint32_t* __restrict__ fwd, int64_t n, int* __restrict__ seen,
                                 int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = fwd[i];
    if (int64_t(v) >= n) {
      atomicOr(bad, 1);
    } else if (atomicAdd(&seen[v], 1) != 0) {
      atomicOr(bad, 1);
    }
  }
}

int bits_for(int64_t extent) {
  int b = 0;
  while ((int64_t(1) << b) < extent) ++b;
  return b;
}

}  // namespace

int order_tokens_impl(int ordering, int64_t f, int64_t h, int64_t w, uint32_t* fwd, uint32_t* inv,
                      int* scratch, int64_t scratch_ints, cudaStream_t stream) {
  Geometry g{};
  g.ordering = ordering;
  g.f = f;
  g.h = h;
  g.w = w;
  switch (ordering) {
    case DFS_RASTER:
      g.virt = f * h * w;
      break;
    case DFS_HILBERT3D: {
      int64_t side = f > h ? f : h;
      side = side > w ? side : w;
      g.bits = bits_for(side);
      if (g.bits > 10) return fail(DFS_E_UNSUPPORTED, "hilbert3d: lattice side > 1024");
      g.virt = int64_t(1) << (3 * g.bits);
      break;
    }
    case DFS_HILBERT2D:
      g.bits = bits_for(h > w ? h : w);
      g.virt = f * (int64_t(1) << (2 * g.bits));
      break;
    case DFS_BLOCK3D:
      g.cf = ceil_div(f, 4);
      g.ch = ceil_div(h, 4);
      g.cw = ceil_div(w, 4);
      g.virt = g.cf * g.ch * g.cw * 64;
      break;
    default:
      return fail(DFS_E_INVALID, "unknown ordering");
  }
  const int64_t nchunks = ceil_div(g.virt, kChunk);
  if (nchunks > scratch_ints) return fail(DFS_E_INTERNAL, "order_tokens: scratch too small");
  count_kernel<<<unsigned(nchunks), kThreads, 0, stream>>>(g, scratch);
  scan_chunks_kernel<<<1, 1024, 0, stream>>>(scratch, int(nchunks));
  write_kernel<<<unsigned(nchunks), kThreads, 0, stream>>>(g, scratch, fwd, inv);
  DFS_LAUNCH_CHECK("order_tokens");
  return DFS_OK;
}

int64_t order_tokens_scratch_ints(int ordering, int64_t f, int64_t h, int64_t w) {
  int64_t virt = f * h * w;
  if (ordering == DFS_HILBERT3D) {
    int64_t side = f > h ? f : h;
    side = side > w ? side : w;
    virt = int64_t(1) << (3 * bits_for(side));
  } else if (ordering == DFS_HILBERT2D) {
    virt = f * (int64_t(1) << (2 * bits_for(h > w ? h : w)));
  } else if (ordering == DFS_BLOCK3D) {
    virt = ceil_div(f, 4) * ceil_div(h, 4) * ceil_div(w, 4) * 64;
  }
  return ceil_div(virt, kChunk) + 1;
}

int invert_permutation_impl(const uint32_t* fwd, int64_t n, uint32_t* inv, cudaStream_t stream) {
  const int64_t blocks = ceil_div(n, 256) < 4 * kNumSMs ? ceil_div(n, 256) : 4 * kNumSMs;
  invert_kernel<<<unsigned(blocks > 0 ? blocks : 1), 256, 0, stream>>>(fwd, n, inv);
  DFS_LAUNCH_CHECK("invert_permutation");
  return DFS_OK;
}

int validate_permutation_impl(const uint32_t* fwd, int64_t n, int* seen, int* bad, int* ok_host,
                              cudaStream_t stream) {
  DFS_CUDA_CHECK(cudaMemsetAsync(seen, 0, sizeof(int) * size_t(n), stream));
  DFS_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), stream));
  const int64_t blocks = ceil_div(n, 256) < 4 * kNumSMs ? ceil_div(n, 256) : 4 * kNumSMs;
  histogram_kernel<<<unsigned(blocks > 0 ? blocks : 1), 256, 0, stream>>>(fwd, n, seen, bad);
  DFS_LAUNCH_CHECK("validate_permutation");
  int hbad = 1;
  DFS_CUDA_CHECK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
  DFS_CUDA_CHECK(cudaStreamSynchronize(stream));
  *ok_host = (hbad == 0 && n > 0) ? 1 : 0;
  return DFS_OK;
}

}  // namespace dfsgpu
