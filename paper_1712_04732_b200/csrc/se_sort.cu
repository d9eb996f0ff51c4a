// Particle binning on the device: stable radix sort of per-particle bin keys
// (CUB), sorted particle records (x, y, z, q) for coalesced reads, bin start
// offsets, and a list of (bin, start, count<=chunk) work units so that heavy
// bins (clustered inputs) are split across CTAs/warps.
//
// Used for the spreading tiles (bins = tiles of stencil start indices) and
// for the real-space cell list (the reference's build_cell_list,
// realspace.py:43-59, which is a stable argsort by cell).
#include <cub/cub.cuh>

#include "se_common.h"

namespace se {

__global__ void iota_kernel(int *a, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int)i;
}

__global__ void gather_records_kernel(const double *__restrict__ pos, const double *__restrict__ q,
                                      const int *__restrict__ idx, double4 *__restrict__ rec, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int j = idx[i];
    rec[i] = make_double4(pos[3 * (int64_t)j], pos[3 * (int64_t)j + 1], pos[3 * (int64_t)j + 2], q ? q[j] : 0.0);
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
                                                           int *__restrict__ nunits, int64_t rlo, int ulo, int uhi) {
    typedef cub::BlockScan<long long, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
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
    Scan(tmp).ExclusiveSum(packed, excl);
    long long cpos = excl >> 32, upos = excl & 0xffffffffLL;
    for (int b = b0; b < b1; ++b) {
        int c = counts[b];
        starts[b] = (int)cpos;
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
        *nunits = (int)upos;
        if (rlo >= cpos) nunits[1] = (int)upos;
        if (rlo < 0 || ulo > 0 || uhi < nbins) nunits[1] = 0;  // no shard start: the list from unit 0
    }
}

int64_t binning_max_units(const Binning &, int64_t N, int nbins, int chunk) {
    return (int64_t)nbins + (N + chunk - 1) / chunk + 1;
}

static int bits_for(int nbins) {
    int b = 1;
    while ((1LL << b) < nbins) ++b;
    return b;
}

void binning_reserve(se_plan *pl, Binning &b, int64_t N, int nbins, int chunk, int extra_bits) {
    int64_t cap = N < 1 ? 1 : N;
    bool grow = cap > b.capacity;
    b.keys.ensure(sizeof(unsigned) * cap);
    b.keys_sorted.ensure(sizeof(unsigned) * cap);
    b.idx_sorted.ensure(sizeof(int) * cap);
    b.rec.ensure(sizeof(double4) * cap);
    if (grow) {
        b.idx.ensure(sizeof(int) * cap);
        // on the plan's stream: the sort that reads idx is ordered after it
        iota_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, pl->stream>>>(b.idx.as<int>(), cap);
        SE_LAUNCH_CHECK();
        b.capacity = cap;
    }
    b.counts.ensure(sizeof(int) * (nbins + 1));
    b.starts.ensure(sizeof(int) * (nbins + 1));
    b.units.ensure(sizeof(int4) * binning_max_units(b, cap, nbins, chunk));
    b.nunits.ensure(sizeof(int) * 2);
    size_t need = 0;
    SE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, b.keys.as<unsigned>(), b.keys_sorted.as<unsigned>(),
                                            b.idx.as<int>(), b.idx_sorted.as<int>(), (int)cap, 0,
                                            bits_for(nbins) + extra_bits));
    b.cub_tmp.ensure(need);
    b.cub_bytes = b.cub_tmp.bytes;
    b.nbins = nbins;
}

// Keys must already be in b.keys and the histogram in b.counts.
void binning_sort(se_plan *pl, Binning &b, const double *pos, const double *q, int64_t N, int nbins, int chunk,
                  int extra_bits, int64_t rlo, int ubin_lo, int ubin_hi) {
    if (ubin_hi < 0) ubin_hi = nbins;
    cudaStream_t st = pl->stream;
    if (N > 0) {
        size_t bytes = b.cub_bytes;
        SE_CUDA(cub::DeviceRadixSort::SortPairs(b.cub_tmp.ptr, bytes, b.keys.as<unsigned>(),
                                                b.keys_sorted.as<unsigned>(), b.idx.as<int>(),
                                                b.idx_sorted.as<int>(), (int)N, 0, bits_for(nbins) + extra_bits,
                                                st));
        gather_records_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(pos, q, b.idx_sorted.as<int>(),
                                                                           b.rec.as<double4>(), N);
        SE_LAUNCH_CHECK();
        pl->launches += 1;
    }
    build_units_kernel<<<1, 1024, 0, st>>>(b.counts.as<int>(), nbins, chunk, b.starts.as<int>(),
                                           b.units.as<int4>(), b.nunits.as<int>(), rlo, ubin_lo, ubin_hi);
    SE_LAUNCH_CHECK();
    pl->launches += 1;
}

}  // namespace se
