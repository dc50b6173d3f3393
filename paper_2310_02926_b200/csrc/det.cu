// det.cu -- deterministic DataBin (bin_spec_t.deterministic = 1).
//
// Atomic accumulation makes fp64 sums depend on update order (PAPER.md:533
// "requires the use of atomic memory updates").  This mode reproduces the
// sequential definition exactly: every bin's sum is folded from +0.0 in
// ascending row order, so results are bit-identical to the oracle (and, with
// nranks > 1, to the oracle's partition mode P = nranks after the
// rank-ordered fold done in handle.cpp).
//
//   k_det_keys      bin index per row (nbins for rows outside the mesh)
//   radix passes    stable LSD sort of (key, row) by key, 8-bit digits:
//                   k_rs_hist -> exclusive scan -> k_rs_scatter
//   k_det_segments  first/last position of every bin in the sorted order
//   k_det_fold      one warp per bin: lanes load 32 consecutive rows, the
//                   fold itself runs in row order through warp shuffles
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"

namespace db {

__device__ __forceinline__ unsigned long long enc_total_d(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    unsigned long long m = (unsigned long long)((long long)b >> 63);
    return b ^ (m | 0x8000000000000000ull);
}

// ---- geometry (same definition as kernels.cu, restated) ----
struct DetGeom {
    double lo[3], scale[3], hi[3];
    int res[3];
    bool ok;
};

__device__ __forceinline__ double dec_total_d(unsigned long long e) {
    unsigned long long m = ~(unsigned long long)((long long)e >> 63);
    return __longlong_as_double((long long)(e ^ (m | 0x8000000000000000ull)));
}

__device__ DetGeom det_geom(const Geom &g, const unsigned long long *bounds) {
    DetGeom G;
    G.ok = true;
    for (int d = 0; d < 3; ++d) {
        G.res[d] = d < g.ndim ? g.res[d] : 1;
        G.lo[d] = 0.0;
        G.hi[d] = 1.0;
        G.scale[d] = 1.0;
        if (d >= g.ndim) continue;
        double lo = g.lo[d], hi = g.hi[d];
        if (g.bounds_auto) {
            unsigned long long elo = bounds[d], nhi = bounds[g.ndim + d];
            if (elo == ~0ull || nhi == ~0ull) G.ok = false;
            lo = dec_total_d(elo);
            hi = dec_total_d(~nhi);
            if (lo == hi) {
                lo = __dsub_rn(lo, 0.5);
                hi = __dadd_rn(hi, 0.5);
            }
            if (!(lo < hi) || isinf(lo) || isinf(hi)) G.ok = false;
        }
        G.lo[d] = lo;
        G.hi[d] = hi;
        G.scale[d] = __ddiv_rn((double)G.res[d], __dsub_rn(hi, lo));
    }
    return G;
}

__global__ void k_det_keys(Geom g, Inputs in, Accum acc, uint32_t *keys, uint32_t *rows) {
    DetGeom G = det_geom(g, acc.bounds);
    const uint32_t B = (uint32_t)acc.nbins;
    uint32_t n_in = 0, n_seen = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < in.n; i += stride) {
        bool inside = G.ok;
        uint32_t b = 0, mul = 1;
        for (int d = 0; d < g.ndim; ++d) {
            double x = in.ax[d][i];
            inside = inside && (G.lo[d] <= x) && (x <= G.hi[d]);
            int kd = min(__double2loint(__dadd_rd(__dmul_rn(__dsub_rn(x, G.lo[d]), G.scale[d]), 4503599627370496.0)), G.res[d] - 1);  // floor (see kernels.cu floor_nonneg)
            b += (uint32_t)kd * mul;
            mul *= (uint32_t)G.res[d];
        }
        keys[i] = inside ? b : B;
        rows[i] = (uint32_t)i;
        n_in += inside;
        n_seen++;
    }
    unsigned long long a = n_in, o = n_seen - n_in;
    for (int s = 16; s > 0; s >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, s);
        o += __shfl_xor_sync(0xffffffffu, o, s);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a) atomicAdd(&acc.count[acc.nbins], a);
        if (o) atomicAdd(&acc.count[acc.nbins + 1], o);
    }
}

// ---- stable LSD radix sort, 8-bit digits, striped tiles of 4096 ----
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t *keys, int64_t n, int shift,
                                                        uint32_t *hist, int64_t nblk) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        int64_t i = base + j * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * nblk + blockIdx.x] = h[threadIdx.x];  // digit-major
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint32_t *keys, const uint32_t *rows, int64_t n,
                                                           int shift, const uint32_t *offs, int64_t nblk,
                                                           uint32_t *keys_out, uint32_t *rows_out) {
    __shared__ uint32_t run[256];
    __shared__ uint32_t wcnt[RS_THREADS / 32][256];
    __shared__ uint32_t base_off[256];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    run[threadIdx.x] = 0;
    base_off[threadIdx.x] = offs[(int64_t)threadIdx.x * nblk + blockIdx.x];
    for (int k = 0; k < RS_THREADS / 32; ++k) wcnt[k][threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    const unsigned lt = (1u << lane) - 1u;
    for (int j = 0; j < RS_ITEMS; ++j) {
        int64_t i = base + j * RS_THREADS + threadIdx.x;
        bool valid = i < n;
        uint32_t key = valid ? keys[i] : 0u, row = valid ? rows[i] : 0u;
        uint32_t d = valid ? ((key >> shift) & 255u) : 256u;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t rank = __popc(peers & lt);
        if (valid && (peers & lt) == 0) wcnt[w][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t pre = run[d];
            for (int k = 0; k < w; ++k) pre += wcnt[k][d];
            uint32_t pos = base_off[d] + pre + rank;
            keys_out[pos] = key;
            rows_out[pos] = row;
        }
        __syncthreads();
        uint32_t add = 0;
        for (int k = 0; k < RS_THREADS / 32; ++k) {
            add += wcnt[k][threadIdx.x];
            wcnt[k][threadIdx.x] = 0;
        }
        run[threadIdx.x] += add;
        __syncthreads();
    }
}

// ---- exclusive scan of u32 (totals < 2^32) ----
constexpr int SC_THREADS = 1024;
constexpr int SC_ITEMS = 4;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t ws[SC_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < SC_THREADS / 32 ? ws[lane] : 0u;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        ws[lane] = s;
    }
    __syncthreads();
    uint32_t pre = (w ? ws[w - 1] : 0u) + x - v;
    *total = ws[SC_THREADS / 32 - 1];
    __syncthreads();
    return pre;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_reduce(const uint32_t *d, int64_t len, uint32_t *part) {
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    uint32_t s = 0;
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + (int64_t)threadIdx.x * SC_ITEMS + k;
        if (i < len) s += d[i];
    }
    uint32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_part(uint32_t *part, int64_t np) {
    uint32_t carry = 0;
    for (int64_t c = 0; c < np; c += SC_THREADS) {
        int64_t i = c + threadIdx.x;
        uint32_t v = i < np ? part[i] : 0u, tot;
        uint32_t pre = block_excl_scan(v, &tot);
        if (i < np) part[i] = carry + pre;
        carry += tot;
    }
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_down(uint32_t *d, int64_t len, const uint32_t *part) {
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    uint32_t v[SC_ITEMS], s = 0;
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + (int64_t)threadIdx.x * SC_ITEMS + k;
        v[k] = i < len ? d[i] : 0u;
        s += v[k];
    }
    uint32_t tot;
    uint32_t pre = block_excl_scan(s, &tot) + part[blockIdx.x];
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + (int64_t)threadIdx.x * SC_ITEMS + k;
        if (i < len) d[i] = pre;
        pre += v[k];
    }
}

static cudaError_t scan_excl(uint32_t *d, int64_t len, uint32_t *part, cudaStream_t s, int *launches) {
    int64_t np = (len + SC_TILE - 1) / SC_TILE;
    if (np == 0) return cudaSuccess;
    k_scan_reduce<<<(unsigned)np, SC_THREADS, 0, s>>>(d, len, part);
    k_scan_part<<<1, SC_THREADS, 0, s>>>(part, np);
    k_scan_down<<<(unsigned)np, SC_THREADS, 0, s>>>(d, len, part);
    *launches += 3;
    return cudaGetLastError();
}

// ---- segments and the in-order fold ----
__global__ void k_det_clear(uint32_t *seg, uint64_t len) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x)
        seg[i] = 0u;
}

__global__ void k_det_segments(const uint32_t *keys, int64_t n, uint32_t B, uint32_t *seg_start, uint32_t *seg_end) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        uint32_t k = keys[j];
        if (k >= B) continue;
        if (j == 0 || keys[j - 1] != k) seg_start[k] = (uint32_t)j;
        if (j == n - 1 || keys[j + 1] != k) seg_end[k] = (uint32_t)(j + 1);
    }
}

__global__ void k_det_fold(Inputs in, Accum acc, const uint32_t *rows, const uint32_t *seg_start,
                           const uint32_t *seg_end) {
    const int lane = threadIdx.x & 31;
    const uint64_t B = acc.nbins;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t b = warp; b < B; b += nwarps) {
        uint32_t j0 = seg_start[b], j1 = seg_end[b];
        if (lane == 0) acc.count[b] = (unsigned long long)(j1 - j0);
        if (j1 == j0) continue;
        for (int a = 0; a < in.nattr; ++a) {
            bool want_sum = (acc.sum_mask >> a) & 1u, want_mm = (acc.mm_mask >> a) & 1u;
            if (!want_sum && !want_mm) continue;
            const double *col = in.at[a];
            double s = 0.0;  // the sequential fold starts at +0.0
            unsigned long long emin = ~0ull, nemax = ~0ull;
            for (uint32_t j = j0; j < j1; j += 32) {
                uint32_t jj = j + lane;
                double v = jj < j1 ? col[rows[jj]] : 0.0;
                int cnt = (int)min(32u, j1 - j);
                if (want_sum)
                    for (int k = 0; k < cnt; ++k) s = __dadd_rn(s, __shfl_sync(0xffffffffu, v, k));
                if (want_mm && jj < j1) {
                    unsigned long long e = enc_total_d(v);
                    emin = e < emin ? e : emin;
                    nemax = ~e < nemax ? ~e : nemax;
                }
            }
            if (want_mm) {
                for (int o = 16; o > 0; o >>= 1) {
                    unsigned long long x = __shfl_xor_sync(0xffffffffu, emin, o);
                    unsigned long long y = __shfl_xor_sync(0xffffffffu, nemax, o);
                    emin = x < emin ? x : emin;
                    nemax = y < nemax ? y : nemax;
                }
            }
            if (lane == 0) {
                if (want_sum) acc.sum[(uint64_t)__popc(acc.sum_mask & ((1u << a) - 1u)) * B + b] = s;
                if (want_mm)
                    ((ulonglong2 *)acc.mm)[(uint64_t)__popc(acc.mm_mask & ((1u << a) - 1u)) * B + b] =
                        make_ulonglong2(emin, nemax);
            }
        }
    }
}

// ---- multi-rank deterministic combine: rank-ordered fold of gathered sums
// (oracle partition mode): s = ((+0.0 + s_0) + s_1) + ...
__global__ void k_det_rank_fold(const double *gathered, int nranks, uint64_t len, double *sum) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s = __dadd_rn(s, gathered[(uint64_t)r * len + i]);
        sum[i] = s;
    }
}

cudaError_t launch_rank_fold(const double *gathered, int nranks, uint64_t len, double *sum, int sms, cudaStream_t s) {
    uint64_t blocks = (len + 255) / 256;
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    if (blocks == 0) return cudaSuccess;
    k_det_rank_fold<<<(unsigned)blocks, 256, 0, s>>>(gathered, nranks, len, sum);
    return cudaGetLastError();
}

// ---- scratch ----
void free_det_scratch(DetScratch &ds) {
    if (ds.device < 0) return;
    DeviceGuard g(ds.device);
    uint32_t *ps[] = {ds.keys, ds.keys_alt, ds.rows, ds.rows_alt, ds.hist, ds.offsets};
    for (uint32_t *p : ps)
        if (p) cudaFree(p);
    if (ds.keys) count_free(ds.cap_rows * 16 + ds.cap_hist * 4 + (int64_t)ds.cap_bins * 8 + 64);
    ds = DetScratch{};
}

int ensure_det_scratch(DetScratch &ds, int64_t n, uint64_t nbins, int device, int sms) {
    (void)sms;
    if (n >= (int64_t)0xffffffffLL) return set_error(BIN_EINVAL, "deterministic mode: %lld rows >= 2^32", (long long)n);
    int64_t nblk = (n + RS_TILE - 1) / RS_TILE;
    int64_t hist_len = 256 * nblk;
    int64_t part_len = (hist_len > (int64_t)nbins + 1 ? hist_len : (int64_t)nbins + 1) / SC_TILE + 2;
    if (ds.keys && ds.device == device && ds.cap_rows >= n && ds.cap_hist >= hist_len + part_len &&
        ds.cap_bins >= nbins)
        return BIN_OK;
    free_det_scratch(ds);
    DeviceGuard g(device);
    int64_t rows = n > 0 ? n : 1;
    ds.device = device;
    ds.cap_rows = rows;
    ds.cap_hist = hist_len + part_len;
    ds.cap_bins = nbins;
    bool ok = cudaMalloc(&ds.keys, rows * 4) == cudaSuccess && cudaMalloc(&ds.keys_alt, rows * 4) == cudaSuccess &&
              cudaMalloc(&ds.rows, rows * 4) == cudaSuccess && cudaMalloc(&ds.rows_alt, rows * 4) == cudaSuccess &&
              cudaMalloc(&ds.hist, ds.cap_hist * 4) == cudaSuccess &&
              cudaMalloc(&ds.offsets, nbins * 8 + 64) == cudaSuccess;
    count_alloc(ds.cap_rows * 16 + ds.cap_hist * 4 + (int64_t)ds.cap_bins * 8 + 64);
    if (!ok) {
        cudaGetLastError();
        free_det_scratch(ds);
        return set_error(BIN_ENOMEM, "deterministic scratch for %lld rows", (long long)n);
    }
    return BIN_OK;
}

cudaError_t launch_deterministic(const Geom &g, const Inputs &in, const Accum &acc, DetScratch &ds,
                                 const LaunchCfg &lc, cudaStream_t s, int *launches) {
    const int64_t n = in.n;
    const uint32_t B = (uint32_t)acc.nbins;
    uint32_t *seg_start = ds.offsets, *seg_end = ds.offsets + acc.nbins;
    int64_t fill_blocks = (int64_t)lc.sms * 8;
    k_det_clear<<<(unsigned)fill_blocks, 256, 0, s>>>(ds.offsets, 2 * acc.nbins);
    (*launches)++;
    if (n > 0) {
        k_det_keys<<<(unsigned)fill_blocks, 256, 0, s>>>(g, in, acc, ds.keys, ds.rows);
        (*launches)++;
        int bits = 0;
        while (bits < 32 && ((uint64_t)B >> bits) != 0) ++bits;  // keys are in [0, B]
        int64_t nblk = (n + RS_TILE - 1) / RS_TILE;
        uint32_t *hist = ds.hist, *part = ds.hist + 256 * nblk;
        uint32_t *k0 = ds.keys, *k1 = ds.keys_alt, *r0 = ds.rows, *r1 = ds.rows_alt;
        for (int shift = 0; shift < bits; shift += 8) {
            k_rs_hist<<<(unsigned)nblk, RS_THREADS, 0, s>>>(k0, n, shift, hist, nblk);
            (*launches)++;
            cudaError_t e = scan_excl(hist, 256 * nblk, part, s, launches);
            if (e != cudaSuccess) return e;
            k_rs_scatter<<<(unsigned)nblk, RS_THREADS, 0, s>>>(k0, r0, n, shift, hist, nblk, k1, r1);
            (*launches)++;
            uint32_t *t = k0; k0 = k1; k1 = t;
            t = r0; r0 = r1; r1 = t;
        }
        k_det_segments<<<(unsigned)fill_blocks, 256, 0, s>>>(k0, n, B, seg_start, seg_end);
        (*launches)++;
        // keep the sorted rows where the fold reads them
        ds.rows_alt = (r0 == ds.rows_alt) ? ds.rows : ds.rows_alt;
        ds.rows = r0;
        ds.keys_alt = (k0 == ds.keys_alt) ? ds.keys : ds.keys_alt;
        ds.keys = k0;
    }
    int64_t fold_blocks = ((int64_t)acc.nbins * 32 + 255) / 256;
    if (fold_blocks > (int64_t)lc.sms * 16) fold_blocks = (int64_t)lc.sms * 16;
    if (fold_blocks < 1) fold_blocks = 1;
    k_det_fold<<<(unsigned)fold_blocks, 256, 0, s>>>(in, acc, ds.rows, seg_start, seg_end);
    (*launches)++;
    return cudaGetLastError();
}

}  // namespace db
