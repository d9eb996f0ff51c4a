// Particle binning on the device: a hand-written counting sort of
// per-particle bin keys (no library sort), sorted particle records
// (x, y, z, q) for coalesced reads, bin start offsets, and a list of
// (bin, start, count<=chunk) work units so that heavy bins (clustered
// inputs) are split across CTAs/warps.
//
// Used for the spreading tiles (bins = tiles of stencil start indices) and
// for the real-space cell list (the reference's build_cell_list,
// realspace.py:43-59, which is a stable argsort by cell).
//
// The sort runs on FINE keys: the real-space key is already fine (column,
// quantized z: the order inside a column must follow z), a tile key is
// refined by the low bits of the particle index.  Each particle takes a
// rank inside its fine bin with one global atomicAdd (fine bins hold ~1
// particle, so the atomics do not contend), the fine histogram is
// exclusive-scanned (three small kernels), the particles are scattered to
// start[key] + rank in ONE pass, and each fine bin's few entries are put in
// index order (an insertion sort per bin): the result is the stable order
// by fine key -- deterministic and identical on every rank that sorts the
// same particles, as the sharded pipeline's contiguous ownership ranges
// require.
#include "se_common.h"

namespace se {

__global__ void iota_kernel(int *a, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int)i;
}

// fine key and rank inside the fine bin
__global__ void fine_rank_kernel(const unsigned *__restrict__ keys, int64_t n, int shift,
                                 unsigned *__restrict__ fkey, int *__restrict__ rank, int *__restrict__ fhist) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned fk = (keys[i] << shift) | ((unsigned)i & ((1u << shift) - 1u));
    fkey[i] = fk;
    rank[i] = atomicAdd(&fhist[fk], 1);
}

// exclusive scan of n ints in three passes: per-block sums, one CTA over
// the block sums, per-block scan plus offset (kScanTile elements per block)
constexpr int kScanThreads = 256, kScanPer = 8, kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ int block_excl_scan(int v, int *sh, int &total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sh[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    total = sh[(blockDim.x >> 5) - 1];
    const int r = x - v + (w ? sh[w - 1] : 0);
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(const int *__restrict__ in, int64_t n,
                                                                 int *__restrict__ bsum) {
    __shared__ int sh[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanPer;
    int s = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) s += base + k < n ? in[base + k] : 0;
    int tot;
    block_excl_scan(s, sh, tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_top_kernel(int *__restrict__ bsum, int nb) {
    __shared__ int sh[32];
    int carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 1024) {
        const int i = b0 + threadIdx.x;
        const int v = i < nb ? bsum[i] : 0;
        int tot;
        const int e = block_excl_scan(v, sh, tot);
        if (i < nb) bsum[i] = carry + e;
        carry += tot;
    }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const int *__restrict__ in, int64_t n,
                                                                  const int *__restrict__ bsum, int *__restrict__ out) {
    __shared__ int sh[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanPer;
    int v[kScanPer], s = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        v[k] = base + k < n ? in[base + k] : 0;
        s += v[k];
    }
    int tot;
    int e = block_excl_scan(s, sh, tot) + bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        if (base + k < n) out[base + k] = e;
        e += v[k];
    }
}

__global__ void scatter_kernel(const unsigned *__restrict__ fkey, const int *__restrict__ rank, int64_t n,
                               const int *__restrict__ fstart, int *__restrict__ idx_sorted) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    idx_sorted[fstart[fkey[i]] + rank[i]] = (int)i;
}

// the entries of each fine bin in index order: an insertion sort per bin
// (bins hold a few particles); bins above kSmallBin entries (coincident z
// layers, extreme clusters) go to a list for bin_order_large_kernel
constexpr int kSmallBin = 48, kLargeBin = 12288;
__global__ void bin_order_kernel(const int *__restrict__ fstart, int64_t nfine, int64_t n, int *__restrict__ idx,
                                 int *__restrict__ large, int *__restrict__ nlarge, int cap) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nfine) return;
    const int s = fstart[b], e = b + 1 < nfine ? fstart[b + 1] : (int)n;
    if (e - s > kSmallBin) {
        const int k = atomicAdd(nlarge, 1);
        if (k < cap) large[k] = (int)b;
        return;
    }
    for (int i = s + 1; i < e; ++i) {
        const int v = idx[i];
        int j = i - 1;
        while (j >= s && idx[j] > v) {
            idx[j + 1] = idx[j];
            --j;
        }
        idx[j + 1] = v;
    }
}

// One CTA per large fine bin: each entry's rank = the number of entries with
// a smaller particle index (the bin in shared memory), written back in
// index order.  Bins beyond kLargeBin entries keep the atomic arrival order
// (correct, not bitwise reproducible); the real-space and spreading work of
// such a bin is quadratic in its size anyway.
__global__ void __launch_bounds__(1024) bin_order_large_kernel(const int *__restrict__ fstart, int64_t nfine, int64_t n,
                                                               int *__restrict__ idx, const int *__restrict__ large,
                                                               const int *__restrict__ nlarge, int cap) {
    __shared__ int v[kLargeBin];
    const int nl = min(*nlarge, cap);
    for (int l = blockIdx.x; l < nl; l += gridDim.x) {
        const int64_t b = large[l];
        const int s = fstart[b], e = b + 1 < nfine ? fstart[b + 1] : (int)n, k = e - s;
        if (k > kLargeBin) continue;
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += blockDim.x) v[i] = idx[s + i];
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += blockDim.x) {
            const int x = v[i];
            int r = 0;
            for (int j = 0; j < k; ++j) r += v[j] < x;
            idx[s + r] = x;
        }
    }
}

__global__ void gather_records_kernel(const double *__restrict__ pos, const double *__restrict__ q,
                                      const int *__restrict__ idx, double4 *__restrict__ rec, int64_t n,
                                      double L) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long j = idx[i];
    rec[i] = make_double4(sane_coord(pos[3 * j], L, j, 0), sane_coord(pos[3 * j + 1], L, j, 1),
                          sane_coord(pos[3 * j + 2], L, j, 2), q ? q[j] : 0.0);
}

// One CTA: exclusive scans of bin counts and of per-bin unit counts, then the
// unit list.  nbins is at most a few 1e5 (tiles or cells), so a single CTA
// with a serial per-thread pass is a few microseconds.
// nunits[0] = number of units; nunits[1] = the unit holding sorted position
// rlo (the first unit of a rank's shard; the unit count if rlo >= N).
// Units are emitted only for bins in [ulo, uhi) (all bins: [0, nbins)); a
// restricted list, or rlo < 0, starts at unit 0 (nunits[1] = 0).
__global__ void __launch_bounds__(1024) build_units_kernel(const int *__restrict__ counts, int nbins, int chunk,
                                                           int *__restrict__ starts, int4 *__restrict__ units,
                                                           int *__restrict__ nunits, int64_t rlo, int ulo, int uhi,
                                                           int *__restrict__ ubstart) {
    __shared__ long long sh[32];
    const int per = (nbins + 1023) / 1024;
    const int b0 = min(nbins, (int)threadIdx.x * per), b1 = min(nbins, b0 + per);
    long long cs = 0, us = 0;
    for (int b = b0; b < b1; ++b) {
        int c = counts[b];
        cs += c;
        if (b >= ulo && b < uhi) us += (c + chunk - 1) / chunk;
    }
    // pack (count prefix, unit prefix) into one 64-bit scan: counts < 2^31, units < 2^31
    long long packed = (cs << 32) | us, excl;
    {   // block-wide exclusive scan of the packed 64-bit pairs
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        long long x = packed;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sh[w] = x;
        __syncthreads();
        if (w == 0) {
            long long s = sh[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            sh[lane] = s;
        }
        __syncthreads();
        excl = x - packed + (w ? sh[w - 1] : 0);
    }
    long long cpos = excl >> 32, upos = excl & 0xffffffffLL;
    for (int b = b0; b < b1; ++b) {
        int c = counts[b];
        starts[b] = (int)cpos;
        ubstart[b] = (int)upos;  // the bin's first unit
        if (b < ulo || b >= uhi) {
            cpos += c;
            continue;
        }
        for (int s = 0; s < c; s += chunk) {
            const int len = min(chunk, c - s);
            if (rlo >= cpos + s && rlo < cpos + s + len) nunits[1] = (int)upos;
            units[upos++] = make_int4(b, (int)cpos + s, len, 0);
        }
        cpos += c;
    }
    if (threadIdx.x == 1023) {
        starts[nbins] = (int)cpos;
        ubstart[nbins] = (int)upos;
        *nunits = (int)upos;
        if (rlo >= cpos) nunits[1] = (int)upos;
        if (rlo < 0 || ulo > 0 || uhi < nbins) nunits[1] = 0;  // no shard start: the list from unit 0
    }
}

int64_t binning_max_units(const Binning &, int64_t N, int nbins, int chunk) {
    return (int64_t)nbins + (N + chunk - 1) / chunk + 1;
}

// index bits that refine a coarse key (tiles): fine bins ~ 4 N at most
static int index_bits(int64_t N, int64_t nfine_coarse) {
    const int64_t cap = std::max<int64_t>(1LL << 20, 4 * N);
    int s = 0;
    while (s < 10 && (nfine_coarse << (s + 1)) <= cap) ++s;
    return s;
}

void binning_reserve(se_plan *pl, Binning &b, int64_t N, int nbins, int chunk, int extra_bits) {
    int64_t cap = N < 1 ? 1 : N;
    b.keys.ensure(sizeof(unsigned) * cap);
    b.keys_sorted.ensure(sizeof(unsigned) * cap);  // fine keys
    b.idx.ensure(sizeof(int) * cap);               // ranks inside the fine bins
    b.idx_sorted.ensure(sizeof(int) * cap);
    b.rec.ensure(sizeof(double4) * cap);
    if (cap > b.capacity) b.capacity = cap;
    b.counts.ensure(sizeof(int) * (nbins + 1));
    b.starts.ensure(sizeof(int) * (nbins + 1));
    b.units.ensure(sizeof(int4) * binning_max_units(b, cap, nbins, chunk));
    b.nunits.ensure(sizeof(int) * 2);
    b.ubstart.ensure(sizeof(int) * (nbins + 1));
    const int64_t coarse = (int64_t)nbins << extra_bits;
    const int shift = extra_bits ? 0 : index_bits(cap, coarse);
    const int64_t nfine = coarse << shift;
    b.fine_shift = shift;
    b.nfine = nfine;
    b.fhist.ensure(sizeof(int) * nfine);
    b.fstart.ensure(sizeof(int) * nfine);
    b.bsum.ensure(sizeof(int) * ((nfine + kScanTile - 1) / kScanTile + 1));
    b.large.ensure(sizeof(int) * (cap / (kSmallBin + 1) + 1));
    b.nlarge.ensure(sizeof(int));
    b.nbins = nbins;
    (void)pl;
}

// Keys must already be in b.keys (bin << extra_bits | sub-key) and the
// coarse histogram in b.counts.
void binning_sort(se_plan *pl, Binning &b, const double *pos, const double *q, int64_t N, int nbins, int chunk,
                  int extra_bits, int64_t rlo, int ubin_lo, int ubin_hi) {
    if (ubin_hi < 0) ubin_hi = nbins;
    cudaStream_t st = pl->stream;
    if (N > 0) {
        const int64_t nfine = b.nfine;
        const unsigned nb = (unsigned)((N + 255) / 256);
        const unsigned fb = (unsigned)((nfine + 255) / 256);
        const unsigned sb = (unsigned)((nfine + kScanTile - 1) / kScanTile);
        SE_CUDA(cudaMemsetAsync(b.fhist.ptr, 0, sizeof(int) * nfine, st));
        fine_rank_kernel<<<nb, 256, 0, st>>>(b.keys.as<unsigned>(), N, b.fine_shift, b.keys_sorted.as<unsigned>(),
                                             b.idx.as<int>(), b.fhist.as<int>());
        scan_sums_kernel<<<sb, kScanThreads, 0, st>>>(b.fhist.as<int>(), nfine, b.bsum.as<int>());
        scan_top_kernel<<<1, 1024, 0, st>>>(b.bsum.as<int>(), (int)sb);
        scan_apply_kernel<<<sb, kScanThreads, 0, st>>>(b.fhist.as<int>(), nfine, b.bsum.as<int>(),
                                                       b.fstart.as<int>());
        scatter_kernel<<<nb, 256, 0, st>>>(b.keys_sorted.as<unsigned>(), b.idx.as<int>(), N, b.fstart.as<int>(),
                                           b.idx_sorted.as<int>());
        SE_CUDA(cudaMemsetAsync(b.nlarge.ptr, 0, sizeof(int), st));
        const int cap = (int)std::min<int64_t>(N / (kSmallBin + 1) + 1, 1 << 20);
        bin_order_kernel<<<fb, 256, 0, st>>>(b.fstart.as<int>(), nfine, N, b.idx_sorted.as<int>(), b.large.as<int>(),
                                             b.nlarge.as<int>(), cap);
        bin_order_large_kernel<<<148, 1024, 0, st>>>(b.fstart.as<int>(), nfine, N, b.idx_sorted.as<int>(),
                                                     b.large.as<int>(), b.nlarge.as<int>(), cap);
        gather_records_kernel<<<nb, 256, 0, st>>>(pos, q, b.idx_sorted.as<int>(), b.rec.as<double4>(), N, pl->L);
        SE_LAUNCH_CHECK();
        pl->launches += 8;
    }
    build_units_kernel<<<1, 1024, 0, st>>>(b.counts.as<int>(), nbins, chunk, b.starts.as<int>(),
                                           b.units.as<int4>(), b.nunits.as<int>(), rlo, ubin_lo, ubin_hi,
                                           b.ubstart.as<int>());
    SE_LAUNCH_CHECK();
    pl->launches += 1;
}

}  // namespace se
