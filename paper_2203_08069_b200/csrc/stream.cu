// Bandwidth-bound leaves and tile plumbing.
//
//  * td_ttv       A(i,j) (+)= sum_k B(i,j,k) c(k)   (reference algorithms.py:280-281)
//  * td_innerprod a (+)= sum B(x) C(x)              (reference algorithms.py:320;
//                 3-order form PAPER.md:1169)
//  * td_copy_box  dst[box] (+)= src[box]           operand assembly, commits
//                 (reference simulator.py:624-634) and send packing
//  * td_fill, td_generate (synthetic inputs; numpy twin oracle/generator.py)
//
// B200 notes: HBM3e is the roof (6.65 TB/s measured copy on this pool).  Rows
// are streamed with 128-bit non-allocating loads (ld.global.nc.L1::no_allocate
// .v2.f64), several in flight per lane; reductions are fixed-order
// (shuffle-xor trees, per-CTA partials then one ordered pass) so results are
// bitwise reproducible run to run.
#include <cstdlib>

#include "common.cuh"

namespace td {

__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream1(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ------------------------------------------------------------------- TTV
// one warp per (i,j) row; VEC: 16-byte aligned rows with even K.
template <bool VEC>
__global__ void __launch_bounds__(256) ttv_kernel(int64_t I, int64_t J, int64_t K, const double* __restrict__ B,
                                                  int64_t sBi, int64_t sBj, const double* __restrict__ c,
                                                  double* __restrict__ A, int64_t sAi, int64_t sAj,
                                                  int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t rows = I * J;
  for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const int64_t i = r / J, j = r - (r / J) * J;
    const double* row = B + i * sBi + j * sBj;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if constexpr (VEC) {
      int64_t k = 2 * lane;
      for (; k + 192 < K; k += 256) {  // four 16-byte loads in flight per lane
        const double2 b0 = ld_stream2(row + k), b1 = ld_stream2(row + k + 64);
        const double2 b2 = ld_stream2(row + k + 128), b3 = ld_stream2(row + k + 192);
        const double2 c0 = *reinterpret_cast<const double2*>(c + k);
        const double2 c1 = *reinterpret_cast<const double2*>(c + k + 64);
        const double2 c2 = *reinterpret_cast<const double2*>(c + k + 128);
        const double2 c3 = *reinterpret_cast<const double2*>(c + k + 192);
        s0 = fma(b0.x, c0.x, s0); s0 = fma(b0.y, c0.y, s0);
        s1 = fma(b1.x, c1.x, s1); s1 = fma(b1.y, c1.y, s1);
        s2 = fma(b2.x, c2.x, s2); s2 = fma(b2.y, c2.y, s2);
        s3 = fma(b3.x, c3.x, s3); s3 = fma(b3.y, c3.y, s3);
      }
      for (; k < K; k += 64) {
        const double2 b0 = ld_stream2(row + k);
        const double2 c0 = *reinterpret_cast<const double2*>(c + k);
        s0 = fma(b0.x, c0.x, s0); s0 = fma(b0.y, c0.y, s0);
      }
    } else {
      for (int64_t k = lane; k < K; k += 32) s0 = fma(ld_stream1(row + k), c[k], s0);
    }
    const double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) {
      double* dst = A + i * sAi + j * sAj;
      *dst = accumulate ? *dst + s : s;
    }
  }
}

// ------------------------------------------------------------- innerprod
constexpr int IP_BLOCKS_PER_SM = 8;
constexpr int IP_THREADS = 256;
constexpr int IP_MAX_BLOCKS = 4096;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// pass 1: the rows x n box is cut into tiles of `chunk` elements; block b owns
// tiles b, b + G, b + 2G, ... so all blocks stream one moving window of HBM
// (DRAM page locality, like TTV's row order) and the assignment stays fixed.
__global__ void __launch_bounds__(IP_THREADS) innerprod_partial(int64_t rows, int64_t n, const double* __restrict__ B,
                                                                int64_t sB, const double* __restrict__ C, int64_t sC,
                                                                double* __restrict__ work, int64_t chunk) {
  __shared__ double sh[32];
  const int64_t total = rows * n;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int64_t t0 = int64_t(blockIdx.x) * chunk; t0 < total; t0 += int64_t(gridDim.x) * chunk) {
  const int64_t e1 = min(total, t0 + chunk);
  for (int64_t e = t0; e < e1;) {
    const int64_t r = e / n;
    const int64_t c0 = e - r * n;
    const int64_t seg = min(n - c0, e1 - e);
    const double* pb = B + r * sB + c0;
    const double* pc = C + r * sC + c0;
    int64_t head = 0;
    const bool same = ((reinterpret_cast<uintptr_t>(pb) ^ reinterpret_cast<uintptr_t>(pc)) & 15) == 0;
    if (same && (reinterpret_cast<uintptr_t>(pb) & 15)) head = 1;
    if (!same) head = seg;
    head = min(head, seg);
    for (int64_t t = threadIdx.x; t < head; t += blockDim.x) a0 = fma(ld_stream1(pb + t), ld_stream1(pc + t), a0);
    const int64_t pairs = (seg - head) / 2;
    const double* vb = pb + head;
    const double* vc = pc + head;
    int64_t q = threadIdx.x;
    for (; q + 3 * IP_THREADS < pairs; q += 4 * IP_THREADS) {
      const double2 b0 = ld_stream2(vb + 2 * q), b1 = ld_stream2(vb + 2 * (q + IP_THREADS));
      const double2 b2 = ld_stream2(vb + 2 * (q + 2 * IP_THREADS)), b3 = ld_stream2(vb + 2 * (q + 3 * IP_THREADS));
      const double2 c0v = ld_stream2(vc + 2 * q), c1v = ld_stream2(vc + 2 * (q + IP_THREADS));
      const double2 c2v = ld_stream2(vc + 2 * (q + 2 * IP_THREADS)), c3v = ld_stream2(vc + 2 * (q + 3 * IP_THREADS));
      a0 = fma(b0.x, c0v.x, a0); a0 = fma(b0.y, c0v.y, a0);
      a1 = fma(b1.x, c1v.x, a1); a1 = fma(b1.y, c1v.y, a1);
      a2 = fma(b2.x, c2v.x, a2); a2 = fma(b2.y, c2v.y, a2);
      a3 = fma(b3.x, c3v.x, a3); a3 = fma(b3.y, c3v.y, a3);
    }
    for (; q < pairs; q += IP_THREADS) {
      const double2 b0 = ld_stream2(vb + 2 * q), c0v = ld_stream2(vc + 2 * q);
      a0 = fma(b0.x, c0v.x, a0); a0 = fma(b0.y, c0v.y, a0);
    }
    const int64_t tail = head + 2 * pairs;
    if (threadIdx.x == 0 && tail < seg) a1 = fma(ld_stream1(pb + tail), ld_stream1(pc + tail), a1);
    e += seg;
  }
  }
  const double s = block_sum((a0 + a1) + (a2 + a3), sh);
  if (threadIdx.x == 0) work[blockIdx.x] = s;
}

// pass 2: fixed-order tree over the partials
// Contiguous operands: the same tiling with the tiles staged by the copy engine
// (cp.async.bulk, one 32 KiB copy per operand per stage, 3-stage mbarrier ring,
// one 512-thread block per SM) -- the SMs issue no global loads at all.  Block
// b owns full tiles b, b + G, ...; block 0 also adds the < IPB_CHUNK tail.
constexpr int IPB_CHUNK = 4096;   // doubles per operand per stage
constexpr int IPB_STAGES = 3;
constexpr int IPB_THREADS = 512;
constexpr int IPB_SMEM = IPB_STAGES * 2 * IPB_CHUNK * 8 + 128;

__device__ __forceinline__ uint32_t ipb_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(IPB_THREADS, 1) innerprod_bulk(int64_t total, const double* __restrict__ B,
                                                                 const double* __restrict__ C,
                                                                 double* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char ipb_raw[];
  __shared__ __align__(8) uint64_t full[IPB_STAGES], empty[IPB_STAGES];
  __shared__ double sh[32];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ipb_raw) + 127) & ~uintptr_t(127));
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t nfull = total / IPB_CHUNK;
  const int64_t G = gridDim.x;
  const int mine = int((nfull - blockIdx.x + G - 1) / G);   // full tiles of this block
  if (tid == 0) {
    for (int s = 0; s < IPB_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(ipb_smem(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(ipb_smem(&empty[s])), "r"(IPB_THREADS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {
    const int s = q % IPB_STAGES;
    const int64_t off = (int64_t(blockIdx.x) + int64_t(q) * G) * IPB_CHUNK;
    const uint32_t bar = ipb_smem(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(2 * IPB_CHUNK * 8)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     ipb_smem(sm + (2 * s) * IPB_CHUNK)),
                 "l"(B + off), "r"(IPB_CHUNK * 8), "r"(bar)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     ipb_smem(sm + (2 * s + 1) * IPB_CHUNK)),
                 "l"(C + off), "r"(IPB_CHUNK * 8), "r"(bar)
                 : "memory");
  };
  auto wait = [](uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                   " selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done)
                   : "r"(ipb_smem(bar)), "r"(parity)
                   : "memory");
    } while (!done);
  };
  if (tid == 0)
    for (int q = 0; q < IPB_STAGES && q < mine; ++q) issue(q);
  double a0 = 0.0, a1 = 0.0;
  for (int q = 0; q < mine; ++q) {
    const int s = q % IPB_STAGES;
    wait(&full[s], (q / IPB_STAGES) & 1);
    const double2* vb = reinterpret_cast<const double2*>(sm + (2 * s) * IPB_CHUNK);
    const double2* vc = reinterpret_cast<const double2*>(sm + (2 * s + 1) * IPB_CHUNK);
#pragma unroll
    for (int i = tid; i < IPB_CHUNK / 2; i += 2 * IPB_THREADS) {
      const double2 b0 = vb[i], c0 = vc[i], b1 = vb[i + IPB_THREADS], c1 = vc[i + IPB_THREADS];
      a0 = fma(b0.x, c0.x, a0);
      a0 = fma(b0.y, c0.y, a0);
      a1 = fma(b1.x, c1.x, a1);
      a1 = fma(b1.y, c1.y, a1);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(ipb_smem(&empty[s])) : "memory");
    if (tid == 0 && q + IPB_STAGES < mine) {
      wait(&empty[s], (q / IPB_STAGES) & 1);   // every warp has read slot s
      issue(q + IPB_STAGES);
    }
  }
  if (blockIdx.x == 0)
    for (int64_t e = nfull * IPB_CHUNK + tid; e < total; e += IPB_THREADS) a1 = fma(B[e], C[e], a1);
  const double sum = block_sum(a0 + a1, sh);
  if (tid == 0) work[blockIdx.x] = sum;
}

// TTV on contiguous rows of K in {512, 1024, 2048, 4096}: tiles of 8192
// doubles (8192 / K whole rows) staged by the copy engine into a 3-stage
// mbarrier ring, c resident in shared memory, 16 warps per block, one block
// per SM.  Warp w sums 512 consecutive elements of one row (lane FMAs +
// shuffle tree) into part[.][w]; the issuing thread, which waits for every
// warp to release a slot before refilling it, adds each row's segment sums in
// ascending order and writes A.
constexpr int TVB_CHUNK = 8192;            // doubles per tile (64 KiB)
constexpr int TVB_STAGES = 3;
constexpr int TVB_EPW = TVB_CHUNK / (IPB_THREADS / 32);   // elements per warp and tile (512)
constexpr int TVB_SMEM = TVB_STAGES * TVB_CHUNK * 8 + 4096 * 8 + 128;

__global__ void __launch_bounds__(IPB_THREADS, 1) ttv_bulk(int64_t rows, int64_t J, int K, const double* __restrict__ B,
                                                           const double* __restrict__ c, double* __restrict__ A,
                                                           int64_t sAi, int64_t sAj, int accumulate) {
  extern __shared__ __align__(128) unsigned char tvb_raw[];
  __shared__ __align__(8) uint64_t full[TVB_STAGES], empty[TVB_STAGES];
  __shared__ double part[2 * TVB_STAGES][IPB_THREADS / 32];   // by q % (2 STAGES): never reused before read
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(tvb_raw) + 127) & ~uintptr_t(127));
  double* cs = sm + TVB_STAGES * TVB_CHUNK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int WARPS = IPB_THREADS / 32;
  const int rpt = TVB_CHUNK / K;            // rows per tile
  const int wpr = WARPS / rpt;              // warps per row
  const int64_t tiles = rows / rpt;
  const int64_t G = gridDim.x;
  const int mine = int((tiles - blockIdx.x + G - 1) / G);
  for (int k = tid; k < K; k += IPB_THREADS) cs[k] = c[k];
  if (tid == 0) {
    for (int s = 0; s < TVB_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(ipb_smem(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(ipb_smem(&empty[s])), "r"(WARPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {
    const int s = q % TVB_STAGES;
    const uint32_t bar = ipb_smem(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(TVB_CHUNK * 8) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     ipb_smem(sm + s * TVB_CHUNK)),
                 "l"(B + (int64_t(blockIdx.x) + int64_t(q) * G) * TVB_CHUNK), "r"(TVB_CHUNK * 8), "r"(bar)
                 : "memory");
  };
  auto wait = [](uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                   " selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done)
                   : "r"(ipb_smem(bar)), "r"(parity)
                   : "memory");
    } while (!done);
  };
  const bool flat = sAi == J * sAj;          // A rows flatten: no division per row
  auto finish = [&](int q) {  // thread 0, after every warp released stage q's slot
    const int pq = q % (2 * TVB_STAGES);
    const int64_t r0 = (int64_t(blockIdx.x) + int64_t(q) * G) * rpt;
    for (int rr = 0; rr < rpt; ++rr) {
      double v = 0.0;
      for (int g = 0; g < wpr; ++g) v += part[pq][rr * wpr + g];
      const int64_t r = r0 + rr;
      double* dst = flat ? A + r * sAj : A + (r / J) * sAi + (r - (r / J) * J) * sAj;
      *dst = accumulate ? *dst + v : v;
    }
  };
  if (tid == 0)
    for (int q = 0; q < TVB_STAGES && q < mine; ++q) issue(q);
  const int row_in_tile = warp / wpr;
  const int k0 = (warp % wpr) * TVB_EPW + 2 * lane;
  for (int q = 0; q < mine; ++q) {
    const int s = q % TVB_STAGES;
    wait(&full[s], (q / TVB_STAGES) & 1);
    const double* rowp = sm + s * TVB_CHUNK + row_in_tile * K;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int u = 0; u < TVB_EPW / 64; u += 2) {
      const double2 b0 = *reinterpret_cast<const double2*>(rowp + k0 + 64 * u);
      const double2 b1 = *reinterpret_cast<const double2*>(rowp + k0 + 64 * (u + 1));
      const double2 c0 = *reinterpret_cast<const double2*>(cs + k0 + 64 * u);
      const double2 c1 = *reinterpret_cast<const double2*>(cs + k0 + 64 * (u + 1));
      s0 = fma(b0.x, c0.x, s0);
      s0 = fma(b0.y, c0.y, s0);
      s1 = fma(b1.x, c1.x, s1);
      s1 = fma(b1.y, c1.y, s1);
    }
    const double w = warp_sum(s0 + s1);
    if (lane == 0) {
      part[q % (2 * TVB_STAGES)][warp] = w;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(ipb_smem(&empty[s])) : "memory");
    }
    if (tid == 0 && q >= 1) {  // the previous stage: every warp is past it by now
      const int p = q - 1;
      wait(&empty[p % TVB_STAGES], (p / TVB_STAGES) & 1);
      if (p + TVB_STAGES < mine) issue(p + TVB_STAGES);
      finish(p);
    }
  }
  if (tid == 0 && mine > 0) {
    const int p = mine - 1;
    wait(&empty[p % TVB_STAGES], (p / TVB_STAGES) & 1);
    finish(p);
  }
}

__global__ void __launch_bounds__(1024) innerprod_final(const double* __restrict__ work, int nparts,
                                                        double* out, int accumulate) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int t = threadIdx.x; t < nparts; t += blockDim.x) v += work[t];
  const double s = block_sum(v, sh);
  if (threadIdx.x == 0) *out = accumulate ? *out + s : s;
}

// ----------------------------------------------------------- box copies
struct BoxArgs {
  int ndim;
  int64_t shape[8];
  int64_t ds[8];
  int64_t ss[8];
};

// rows = product of all but the last axis; one block-stride loop per row
__global__ void __launch_bounds__(256) copy_box_kernel(BoxArgs a, double* dst, const double* src, int64_t rows,
                                                       int accumulate) {
  const int nd = a.ndim;
  const int64_t inner = a.shape[nd - 1];
  const int64_t dsi = a.ds[nd - 1], ssi = a.ss[nd - 1];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    int64_t rem = r, doff = 0, soff = 0;
    for (int d = nd - 2; d >= 0; --d) {
      const int64_t q = rem / a.shape[d];
      const int64_t c = rem - q * a.shape[d];
      rem = q;
      doff += c * a.ds[d];
      soff += c * a.ss[d];
    }
    double* drow = dst + doff;
    const double* srow = src + soff;
    if (accumulate) {
      for (int64_t x = threadIdx.x; x < inner; x += blockDim.x) drow[x * dsi] += srow[x * ssi];
    } else {
      for (int64_t x = threadIdx.x; x < inner; x += blockDim.x) drow[x * dsi] = srow[x * ssi];
    }
  }
}

__global__ void fill_kernel(double* dst, int64_t n, double v) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    dst[e] = v;
}

// ----------------------------------------------------------- generator
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct GenArgs {
  int ndim;
  int64_t gstride[8];  // global row-major strides
  int64_t origin[8];
  int64_t shape[8];
  int64_t ds[8];
  uint64_t key;
  int mode;
};

__global__ void __launch_bounds__(256) generate_kernel(GenArgs a, double* dst, int64_t total) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = e, g = 0, off = 0;
    for (int d = a.ndim - 1; d >= 0; --d) {
      const int64_t q = rem / a.shape[d];
      const int64_t c = rem - q * a.shape[d];
      rem = q;
      g += (a.origin[d] + c) * a.gstride[d];
      off += c * a.ds[d];
    }
    const uint64_t h = splitmix64(a.key ^ uint64_t(g));
    double v;
    if (a.mode == 0) v = double(int64_t(h % 9ull) - 4);
    else v = double(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    dst[off] = v;
  }
}

}  // namespace td

extern "C" {

int td_ttv(void* stream, int64_t I, int64_t J, int64_t K, const double* B, int64_t sBi, int64_t sBj,
           const double* c, double* A, int64_t sAi, int64_t sAj, int accumulate) {
  using namespace td;
  if (I <= 0 || J <= 0) return TD_OK;
  StreamDevice sd(stream);
  const int64_t rows = I * J;
  const bool vec = K % 2 == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(c) & 15) == 0 && sBi % 2 == 0 && sBj % 2 == 0;
  const int64_t want = ceil_div(rows, 8);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * 8));
  static const bool bulk_on = [] {
    const char* e = std::getenv("TD_TTV_BULK");
    return e == nullptr || std::atoi(e) != 0;
  }();
  const bool rows_contiguous = sBj == K && (I == 1 || sBi == J * K);
  if (bulk_on && vec && rows_contiguous && K >= TVB_EPW && K <= 4096 && TVB_CHUNK % K == 0 &&
      rows % (TVB_CHUNK / K) == 0 && rows / (TVB_CHUNK / K) >= 4 * num_sms() &&
      (reinterpret_cast<uintptr_t>(c) & 15) == 0) {
    TD_CUDA(ensure_smem(ttv_bulk, TVB_SMEM));
    ttv_bulk<<<num_sms(), IPB_THREADS, TVB_SMEM, as_stream(stream)>>>(rows, J, (int)K, B, c, A, sAi, sAj, accumulate);
    return check_launch("ttv_bulk");
  }
  if (vec) ttv_kernel<true><<<blocks, 256, 0, as_stream(stream)>>>(I, J, K, B, sBi, sBj, c, A, sAi, sAj, accumulate);
  else ttv_kernel<false><<<blocks, 256, 0, as_stream(stream)>>>(I, J, K, B, sBi, sBj, c, A, sAi, sAj, accumulate);
  return check_launch("ttv_kernel");
}

int64_t td_innerprod_work_size(void) { return td::IP_MAX_BLOCKS; }

int td_innerprod(void* stream, int64_t rows, int64_t n, const double* B, int64_t sB, const double* C, int64_t sC,
                 double* out, double* work, int accumulate) {
  using namespace td;
  StreamDevice sd(stream);
  cudaStream_t st = as_stream(stream);
  const int64_t total = rows > 0 && n > 0 ? rows * n : 0;
  int parts = (int)std::min<int64_t>((int64_t)num_sms() * IP_BLOCKS_PER_SM, IP_MAX_BLOCKS);
  // 8192-element tiles (64 KiB per operand), interleaved over the blocks
  const int64_t chunk = 8192;
  parts = (int)std::max<int64_t>(1, std::min<int64_t>(parts, ceil_div(total, chunk)));
  static const bool bulk_on = [] {
    const char* e = std::getenv("TD_IP_BULK");
    return e == nullptr || std::atoi(e) != 0;
  }();
  const bool contiguous = (rows == 1 || (sB == n && sC == n)) && (reinterpret_cast<uintptr_t>(B) & 15) == 0 &&
                          (reinterpret_cast<uintptr_t>(C) & 15) == 0;
  if (bulk_on && contiguous && total >= int64_t(IPB_CHUNK) * num_sms()) {
    parts = num_sms();
    TD_CUDA(ensure_smem(innerprod_bulk, IPB_SMEM));
    innerprod_bulk<<<parts, IPB_THREADS, IPB_SMEM, st>>>(total, B, C, work);
    if (int rc = check_launch("innerprod_bulk")) return rc;
  } else if (total > 0) {
    innerprod_partial<<<parts, IP_THREADS, 0, st>>>(rows, n, B, sB, C, sC, work, chunk);
    int rc = check_launch("innerprod_partial");
    if (rc) return rc;
  } else {
    parts = 0;
  }
  innerprod_final<<<1, 1024, 0, st>>>(work, parts, out, accumulate);
  return check_launch("innerprod_final");
}

int td_copy_box(void* stream, int ndim, const int64_t* shape, double* dst, const int64_t* dst_strides,
                const double* src, const int64_t* src_strides, int accumulate) {
  using namespace td;
  TD_REQUIRE(ndim >= 0 && ndim <= 8, "copy_box: ndim %d out of range", ndim);
  StreamDevice sd(stream);
  BoxArgs a{};
  int64_t vol = 1;
  if (ndim == 0) {  // scalar
    a.ndim = 1;
    a.shape[0] = 1;
    a.ds[0] = a.ss[0] = 1;
  } else {
    a.ndim = ndim;
    for (int d = 0; d < ndim; ++d) {
      a.shape[d] = shape[d];
      a.ds[d] = dst_strides[d];
      a.ss[d] = src_strides[d];
      vol *= shape[d];
    }
  }
  if (vol <= 0) return TD_OK;
  const int64_t rows = vol / a.shape[a.ndim - 1];
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)num_sms() * 16));
  copy_box_kernel<<<blocks, 256, 0, as_stream(stream)>>>(a, dst, src, rows, accumulate);
  return check_launch("copy_box_kernel");
}

int td_fill(void* stream, double* dst, int64_t n, double value) {
  using namespace td;
  if (n <= 0) return TD_OK;
  StreamDevice sd(stream);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 16));
  fill_kernel<<<blocks, 256, 0, as_stream(stream)>>>(dst, n, value);
  return check_launch("fill_kernel");
}

int td_generate(void* stream, int ndim, const int64_t* gdims, const int64_t* origin, const int64_t* shape,
                double* dst, const int64_t* dst_strides, uint64_t seed, uint64_t tensor_id, int mode) {
  using namespace td;
  TD_REQUIRE(ndim >= 0 && ndim <= 8, "generate: ndim %d out of range", ndim);
  StreamDevice sd(stream);
  GenArgs a{};
  int64_t total = 1;
  if (ndim == 0) {
    a.ndim = 1;
    a.gstride[0] = 1;
    a.shape[0] = 1;
    a.ds[0] = 1;
  } else {
    a.ndim = ndim;
    int64_t st = 1;
    for (int d = ndim - 1; d >= 0; --d) {
      a.gstride[d] = st;
      st *= gdims[d];
    }
    for (int d = 0; d < ndim; ++d) {
      a.origin[d] = origin[d];
      a.shape[d] = shape[d];
      a.ds[d] = dst_strides[d];
      total *= shape[d];
    }
  }
  a.key = splitmix64(splitmix64(seed) ^ (tensor_id * 0xD1B54A32D192ED03ull));
  a.mode = mode;
  if (total <= 0) return TD_OK;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 16));
  generate_kernel<<<blocks, 256, 0, as_stream(stream)>>>(a, dst, total);
  return check_launch("generate_kernel");
}

}  // extern "C"
