// Microbenchmarks that decide the DataBin accumulate design on sm_100a
// (SURVEY.md §7 step 5). Not product code: a standalone executable.
//
// Measures, for uniform-random and hot-spot ("Plummer-like") address
// streams:
//   * shared-memory atomics: u32 add, f64 add (CAS loop), u64 min (CAS),
//     and plain (racy) LDS+STS read-modify-write as the ceiling;
//   * global (L2) REDs: u32 add, u64 add, f64 add, u64 min, pairs;
//   * random L2 loads (the min/max "filter" read);
//   * DSMEM red.shared::cluster.add.u32 / f64 at cluster size 8 and 16;
//   * HBM streaming read bandwidth with 128-bit loads;
//   * MATCH.ANY cost.
// Output: one JSON object per line on stdout.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo \
//        -o atomics_bench atomics_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
// pattern 0: uniform over nbins; pattern 1: half the ops hit a hot set of 800 bins
__device__ __forceinline__ uint32_t pick(uint32_t h, uint32_t nbins, int pattern) {
  if (pattern == 1 && (h & 0x80000000u)) return (h >> 8) % 800u;
  return h % nbins;
}

constexpr int ITERS = 64;

// ---------------- shared memory ----------------
template <int OP>
__global__ void k_smem(uint32_t nbins, int pattern, unsigned long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint32_t* s32 = (uint32_t*)sm; double* sf = (double*)sm; unsigned long long* s64 = (unsigned long long*)sm;
  int words = (OP == 0) ? nbins : nbins * 2;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s32[i] = 0;
  __syncthreads();
  uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * ITERS;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    uint32_t h = hash32(base + i);
    uint32_t b = pick(h, nbins, pattern);
    if (OP == 0) atomicAdd(&s32[b], h & 7);
    else if (OP == 1) atomicAdd(&sf[b], (double)(h & 1023));
    else if (OP == 2) atomicMin(&s64[b], (unsigned long long)h);
    else if (OP == 3) { double v = sf[b]; sf[b] = v + (double)(h & 1023); }
    else if (OP == 4) { // min filter: load then CAS only if improving
      unsigned long long v = h; if (v < s64[b]) atomicMin(&s64[b], v);
    }
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) acc += s32[i];
  if (acc == 0x1234567) out[0] = acc;  // defeat DCE
}

// ---------------- global (L2 / HBM) ----------------
template <int OP>
__global__ void k_gmem(void* g, uint32_t nbins, int pattern, unsigned long long* out) {
  uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * ITERS;
  unsigned long long acc = 0;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    uint32_t h = hash32(base + i);
    uint32_t b = pick(h, nbins, pattern);
    if (OP == 0) atomicAdd(&((uint32_t*)g)[b], 1u);
    else if (OP == 1) atomicAdd(&((unsigned long long*)g)[b], 1ull);
    else if (OP == 2) atomicAdd(&((double*)g)[b], (double)(h & 1023));
    else if (OP == 3) atomicMin(&((unsigned long long*)g)[b], (unsigned long long)h);
    else if (OP == 4) { // count u64 + f64 sum in one 16 B record
      atomicAdd(&((unsigned long long*)g)[2 * b], 1ull);
      atomicAdd(&((double*)g)[2 * b + 1], (double)(h & 1023));
    } else if (OP == 5) { acc += __ldcg(&((const unsigned long long*)g)[b]); }
    else if (OP == 6) { // 32 B record: count, sum, filtered min/max via one 16 B load
      unsigned long long* r = &((unsigned long long*)g)[4 * b];
      atomicAdd(&r[0], 1ull);
      atomicAdd((double*)&r[1], (double)(h & 1023));
      ulonglong2 mm = __ldcg((const ulonglong2*)&r[2]);
      unsigned long long v = h;
      if (v < mm.x) atomicMin(&r[2], v);
      if (v > mm.y) atomicMax(&r[3], v);
    }
  }
  if (acc == 0x1234567) out[0] = acc;
}

// ---------------- DSMEM ----------------
template <int OP>
__global__ void k_dsmem(uint32_t nbins_per_cta, int pattern, unsigned long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  uint32_t* s32 = (uint32_t*)sm; double* sf = (double*)sm;
  int words = (OP == 0) ? nbins_per_cta : nbins_per_cta * 2;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s32[i] = 0;
  cl.sync();
  unsigned csize = cl.num_blocks();
  uint32_t total = nbins_per_cta * csize;
  uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * ITERS;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    uint32_t h = hash32(base + i);
    uint32_t b = pick(h, total, pattern);
    unsigned rank = b / nbins_per_cta, off = b % nbins_per_cta;
    if (OP == 0) {
      uint32_t* p = cl.map_shared_rank(s32, rank);
      atomicAdd(p + off, 1u);
    } else {
      double* p = cl.map_shared_rank(sf, rank);
      atomicAdd(p + off, (double)(h & 1023));
    }
  }
  cl.sync();
  unsigned long long acc = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) acc += s32[i];
  if (acc == 0x1234567) out[0] = acc;
}

// ---------------- HBM stream read ----------------
__global__ void k_stream(const double2* __restrict__ p, size_t n2, unsigned long long* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
    acc += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
  }
  for (; i < n2; i += stride) { double2 a = __ldcs(p + i); acc += a.x + a.y; }
  if (acc == 1.2345) out[0] = 1;
}

__global__ void k_match(int pattern, unsigned long long* out) {
  uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * ITERS;
  unsigned acc = 0;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    uint32_t h = hash32(base + i);
    uint32_t b = pick(h, 262144, pattern);
    acc += __match_any_sync(0xffffffffu, b);
  }
  if (acc == 0x1234567) out[0] = acc;
}

static float time_launch(void (*launch)(void*), void* ctx, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  launch(ctx); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); launch(ctx); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

struct Ctx { int grid, block, smem, pattern, op, cluster; uint32_t nbins; void* g; unsigned long long* out; const double2* p; size_t n2; };

template <int OP> static void L_smem(void* c_) { Ctx* c = (Ctx*)c_; k_smem<OP><<<c->grid, c->block, c->smem>>>(c->nbins, c->pattern, c->out); }
template <int OP> static void L_gmem(void* c_) { Ctx* c = (Ctx*)c_; k_gmem<OP><<<c->grid, c->block>>>(c->g, c->nbins, c->pattern, c->out); }
template <int OP> static void L_dsmem(void* c_) {
  Ctx* c = (Ctx*)c_;
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(c->grid); cfg.blockDim = dim3(c->block); cfg.dynamicSmemBytes = c->smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = c->cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_dsmem<OP>, c->nbins, c->pattern, c->out));
}
static void L_stream(void* c_) { Ctx* c = (Ctx*)c_; k_stream<<<c->grid, c->block>>>(c->p, c->n2, c->out); }
static void L_match(void* c_) { Ctx* c = (Ctx*)c_; k_match<<<c->grid, c->block>>>(c->pattern, c->out); }

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int nsm = prop.multiProcessorCount;
  printf("{\"device\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu,\"clock_khz\":%d}\n",
         prop.name, nsm, prop.l2CacheSize, prop.sharedMemPerBlockOptin, prop.clockRate);
  unsigned long long* out; CK(cudaMalloc(&out, 64));
  const char* pat[2] = {"uniform", "hot"};
  // shared-memory atomics
  const char* sname[5] = {"smem_u32_add", "smem_f64_add_cas", "smem_u64_min", "smem_f64_plain_rmw", "smem_u64_min_filtered"};
  void (*sl[5])(void*) = {L_smem<0>, L_smem<1>, L_smem<2>, L_smem<3>, L_smem<4>};
  for (int op = 0; op < 5; ++op) {
    uint32_t nb_list[2] = {4096, 16384};
    for (uint32_t nb : nb_list) for (int pt = 0; pt < 2; ++pt) for (int bs : {256, 512}) {
      Ctx c{}; c.block = bs; c.nbins = nb; c.pattern = pt;
      c.smem = (op == 0 ? 4 : 8) * nb; c.out = out;
      int occ = 0;
      if (op == 0) { CK(cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000)); CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_smem<0>, bs, c.smem)); }
      if (op == 1) { CK(cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000)); CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_smem<1>, bs, c.smem)); }
      if (op == 2) { CK(cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000)); CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_smem<2>, bs, c.smem)); }
      if (op == 3) { CK(cudaFuncSetAttribute(k_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000)); CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_smem<3>, bs, c.smem)); }
      if (op == 4) { CK(cudaFuncSetAttribute(k_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000)); CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_smem<4>, bs, c.smem)); }
      c.grid = nsm * occ * 8;
      float ms = time_launch(sl[op], &c);
      double ops = (double)c.grid * bs * ITERS;
      printf("{\"test\":\"%s\",\"nbins\":%u,\"pattern\":\"%s\",\"block\":%d,\"occ\":%d,\"ms\":%.4f,\"Gops\":%.2f,\"ops_per_sm_clk_at_1.9GHz\":%.3f}\n",
             sname[op], nb, pat[pt], bs, occ, ms, ops / ms / 1e6, ops / ms / 1e6 / nsm / 1.9);
    }
  }
  // global
  void* g; size_t gbytes = (size_t)1 << 31; CK(cudaMalloc(&g, gbytes));
  const char* gname[7] = {"g_u32_add", "g_u64_add", "g_f64_add", "g_u64_min", "g_pair_cnt_sum", "g_ld_random", "g_rec32_full"};
  void (*gl[7])(void*) = {L_gmem<0>, L_gmem<1>, L_gmem<2>, L_gmem<3>, L_gmem<4>, L_gmem<5>, L_gmem<6>};
  for (int op = 0; op < 7; ++op) {
    uint32_t nb_list[3] = {65536, 262144, 16777216};
    for (uint32_t nb : nb_list) for (int pt = 0; pt < 2; ++pt) {
      CK(cudaMemset(g, 0, (size_t)nb * 32));
      Ctx c{}; c.block = 256; c.nbins = nb; c.pattern = pt; c.g = g; c.out = out; c.grid = nsm * 8 * 16;
      float ms = time_launch(gl[op], &c);
      double ops = (double)c.grid * c.block * ITERS;
      printf("{\"test\":\"%s\",\"nbins\":%u,\"pattern\":\"%s\",\"ms\":%.4f,\"Gops\":%.2f,\"ops_per_sm_clk_at_1.9GHz\":%.3f}\n",
             gname[op], nb, pat[pt], ms, ops / ms / 1e6, ops / ms / 1e6 / nsm / 1.9);
    }
  }
  // DSMEM
  CK(cudaFuncSetAttribute(k_dsmem<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_dsmem<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_dsmem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
  CK(cudaFuncSetAttribute(k_dsmem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
  for (int op = 0; op < 2; ++op) for (int cs : {2, 8, 16}) for (int pt = 0; pt < 2; ++pt) {
    Ctx c{}; c.block = 512; c.nbins = 16384; c.pattern = pt; c.out = out; c.cluster = cs;
    c.smem = (op == 0 ? 4 : 8) * c.nbins; c.grid = (nsm / cs) * cs * 4;
    float ms = time_launch(op == 0 ? L_dsmem<0> : L_dsmem<1>, &c);
    cudaError_t e = cudaGetLastError();
    double ops = (double)c.grid * c.block * ITERS;
    printf("{\"test\":\"%s\",\"cluster\":%d,\"pattern\":\"%s\",\"ms\":%.4f,\"Gops\":%.2f,\"err\":\"%s\"}\n",
           op == 0 ? "dsmem_u32_add" : "dsmem_f64_add", cs, pat[pt], ms, ops / ms / 1e6, cudaGetErrorString(e));
  }
  // stream
  {
    size_t bytes = (size_t)2400 * 1000 * 1000; double2* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes));
    for (int mult : {2, 4, 8, 16}) for (int bs : {256, 512}) {
      Ctx c{}; c.block = bs; c.grid = nsm * mult; c.p = p; c.n2 = bytes / 16; c.out = out;
      float ms = time_launch(L_stream, &c);
      printf("{\"test\":\"hbm_stream_read\",\"grid\":%d,\"block\":%d,\"ms\":%.4f,\"GBps\":%.1f}\n", c.grid, bs, ms, bytes / ms / 1e6);
    }
    CK(cudaFree(p));
  }
  for (int pt = 0; pt < 2; ++pt) {
    Ctx c{}; c.block = 256; c.grid = nsm * 8 * 16; c.pattern = pt; c.out = out;
    float ms = time_launch(L_match, &c);
    double ops = (double)c.grid * c.block * ITERS;
    printf("{\"test\":\"match_any\",\"pattern\":\"%s\",\"ms\":%.4f,\"Glane_ops\":%.2f,\"warp_ops_per_sm_clk\":%.3f}\n",
           pat[pt], ms, ops / ms / 1e6, ops / 32 / ms / 1e6 / nsm / 1.9);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
