// Real-space Ewald sum and self term: realspace.real_space_sum /
// realspace.self_term (realspace.py:91-185).
//
// phi_R(x_t) = sum_{s, image p, |x_t - x_s + p| < rc, r >= 1e-14} q_s erfc(xi r)/r
//
// Cell path (rc <= L/2 on periodic axes, or any rc for free axes):
//  * cells of edge >= rc/2 (n = floor(2L/rc) per axis, vs the reference's
//    rc-edge cells): the 5x5x5 neighbourhood covers the cutoff sphere with
//    ~3.7x fewer candidates per target than 3x3x3 rc-cells;
//  * particles stable-sorted by cell (the reference's build_cell_list,
//    realspace.py:43-59) into (x, y, z, q) double4 records;
//  * one warp per (cell, <=32 targets) unit; sources are streamed through a
//    per-warp shared-memory stage (32 records) with the periodic image shift
//    folded in once per source run, so the pair test is 3 sub + 3 mul/fma;
//  * neighbour cells are visited as contiguous z-runs of the sorted order;
//    periodic axes with fewer than 5 cells visit every cell once and use the
//    minimum image per pair (the reference's (cell, shift) de-duplication for
//    n <= 2, realspace.py:98-109, gives the same pair set).
// Image path (D >= 1 and rc > L/2): all pairs x explicit images
// (realspace.py:138-165), one thread per target.
#include "se_common.h"

namespace se {

struct RealArgs {
    int n;           // cells per axis
    double edge, L, xi, rc, rc2;
    int mode[3];     // 0 free, 1 periodic +-2 wrap, 2 periodic all cells + min image
    int64_t rlo, rhi;
    int add_self;
    double self_coef;  // -2 xi / sqrt(pi) applied as ((-2 xi) q) / sqrt(pi)
    double sqrtpi;
};

__global__ void cell_keys_kernel(const double *__restrict__ pos, int64_t N, RealArgs a, unsigned *__restrict__ keys,
                                 int *__restrict__ counts) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int c[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        int ci = (int)(pos[3 * i + ax] / a.edge);
        c[ax] = ci < a.n - 1 ? ci : a.n - 1;
    }
    unsigned key = (unsigned)((c[0] * a.n + c[1]) * a.n + c[2]);
    keys[i] = key;
    atomicAdd(&counts[key], 1);
}

__device__ __forceinline__ double min_image(double d, double L) { return d - L * rint(d / L); }

template <bool MI, bool COUNT>
__device__ __forceinline__ void pair_run(const double4 *__restrict__ rec, int j0, int j1, double shx, double shy,
                                         double shz, const RealArgs &a, double4 *st, int *sj, double4 tp, int tidx,
                                         bool active, double &acc, int &singular, const int mi[3], long long &cnt) {
    const int lane = threadIdx.x & 31;
    for (int jb = j0; jb < j1; jb += 32) {
        int j = jb + lane;
        if (j < j1) {
            double4 r = rec[j];
            st[lane] = make_double4(__dadd_rn(r.x, shx), __dadd_rn(r.y, shy), __dadd_rn(r.z, shz), r.w);
            sj[lane] = j;
        }
        __syncwarp();
        int m = min(32, j1 - jb);
        if (active) {
            for (int k = 0; k < m; ++k) {
                double4 s = st[k];
                double dx = __dsub_rn(tp.x, s.x), dy = __dsub_rn(tp.y, s.y), dz = __dsub_rn(tp.z, s.z);
                if (MI) {
                    if (mi[0]) dx = min_image(dx, a.L);
                    if (mi[1]) dy = min_image(dy, a.L);
                    if (mi[2]) dz = min_image(dz, a.L);
                }
                double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                if (r2 < a.rc2) {
                    double r = sqrt(r2);
                    if (r < a.rc) {
                        if (r < 1e-14) {
                            if (sj[k] != tidx) singular = 1;
                        } else if (COUNT) {
                            ++cnt;
                        } else {
                            acc += s.w * (erfc(a.xi * r) / r);
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
}

template <bool MI, bool COUNT>
__global__ void __launch_bounds__(128) realspace_cell_kernel(const double4 *__restrict__ rec, const int *__restrict__ sidx,
                                                             const int *__restrict__ starts, const int4 *__restrict__ units,
                                                             const int *__restrict__ nunits, RealArgs a,
                                                             double *__restrict__ phi, int *__restrict__ flag,
                                                             unsigned long long *__restrict__ npairs) {
    __shared__ double4 stage[4][32];
    __shared__ int sj[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int u = blockIdx.x * 4 + warp;
    if (u >= *nunits) return;
    int4 un = units[u];
    const int n = a.n;
    const int cell = un.x;
    const int cz = cell % n, cy = (cell / n) % n, cx = cell / (n * n);
    int t = un.y + lane;
    bool active = lane < un.z && t >= a.rlo && t < a.rhi;
    if (__ballot_sync(0xffffffffu, active) == 0) return;
    double4 tp = active ? rec[t] : make_double4(0, 0, 0, 0);
    double acc = 0.0;
    int singular = 0;
    long long cnt = 0;
    const int mi[3] = {a.mode[0] == 2, a.mode[1] == 2, a.mode[2] == 2};

    // per-axis candidate lists: (cell, shift index) for x and y; z as runs
    int xs_lo, xs_hi, ys_lo, ys_hi;
    auto axis_range = [&](int c, int mode, int &lo, int &hi) {
        if (mode == 2) {
            lo = 0;
            hi = n - 1;
        } else if (mode == 1) {
            lo = c - 2;
            hi = c + 2;
        } else {
            lo = max(0, c - 2);
            hi = min(n - 1, c + 2);
        }
    };
    axis_range(cx, a.mode[0], xs_lo, xs_hi);
    axis_range(cy, a.mode[1], ys_lo, ys_hi);
    int zlo, zhi;
    axis_range(cz, a.mode[2], zlo, zhi);
    for (int ox = xs_lo; ox <= xs_hi; ++ox) {
        int xc = ox;
        double shx = 0.0;
        if (a.mode[0] == 1) {
            if (xc < 0) { xc += n; shx = -a.L; }
            else if (xc >= n) { xc -= n; shx = a.L; }
        }
        for (int oy = ys_lo; oy <= ys_hi; ++oy) {
            int yc = oy;
            double shy = 0.0;
            if (a.mode[1] == 1) {
                if (yc < 0) { yc += n; shy = -a.L; }
                else if (yc >= n) { yc -= n; shy = a.L; }
            }
            const int rowbase = (xc * n + yc) * n;
            if (a.mode[2] == 1) {
                // up to three runs: wrapped below, in range, wrapped above
                int r0 = zlo, r1 = zhi;
                int blo = max(r0, 0), bhi = min(r1, n - 1);
                if (r0 < 0) {
                    int c0 = r0 + n, c1 = n - 1;
                    pair_run<MI, COUNT>(rec, starts[rowbase + c0], starts[rowbase + c1 + 1], shx, shy, -a.L, a, stage[warp],
                                 sj[warp], tp, t, active, acc, singular, mi, cnt);
                }
                if (blo <= bhi)
                    pair_run<MI, COUNT>(rec, starts[rowbase + blo], starts[rowbase + bhi + 1], shx, shy, 0.0, a, stage[warp],
                                 sj[warp], tp, t, active, acc, singular, mi, cnt);
                if (r1 > n - 1) {
                    int c0 = 0, c1 = r1 - n;
                    pair_run<MI, COUNT>(rec, starts[rowbase + c0], starts[rowbase + c1 + 1], shx, shy, a.L, a, stage[warp],
                                 sj[warp], tp, t, active, acc, singular, mi, cnt);
                }
            } else {
                pair_run<MI, COUNT>(rec, starts[rowbase + zlo], starts[rowbase + zhi + 1], shx, shy, 0.0, a, stage[warp],
                             sj[warp], tp, t, active, acc, singular, mi, cnt);
            }
        }
    }
    if (COUNT) {
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) atomicAdd(npairs, (unsigned long long)cnt);
        return;
    }
    if (active) {
        if (singular) atomicExch(flag, 1);
        double v = acc;
        if (a.add_self) v += (-2.0 * a.xi * tp.w) / a.sqrtpi;
        phi[sidx[t]] = v;
    }
}

// rc > L/2 with periodic axes: explicit images (realspace.py:138-165)
__global__ void realspace_image_kernel(const double *__restrict__ pos, const double *__restrict__ q, int64_t N,
                                       int64_t rlo, int64_t rhi, RealArgs a, int D, int layers,
                                       double *__restrict__ phi, int *__restrict__ flag) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N) return;
    bool own = t >= rlo && t < rhi;
    if (!own) return;
    double xt = pos[3 * t], yt = pos[3 * t + 1], zt = pos[3 * t + 2];
    int lx = D >= 1 ? layers : 0, ly = D >= 2 ? layers : 0, lz = D >= 3 ? layers : 0;
    double acc = 0.0;
    int err = 0;
    for (int ax = -lx; ax <= lx; ++ax)
        for (int ay = -ly; ay <= ly; ++ay)
            for (int az = -lz; az <= lz; ++az) {
                double sx = ax * a.L, sy = ay * a.L, sz = az * a.L;
                bool origin = ax == 0 && ay == 0 && az == 0;
                double img = 0.0;
                for (int64_t s = 0; s < N; ++s) {
                    double dx = __dadd_rn(__dsub_rn(xt, pos[3 * s]), sx);
                    double dy = __dadd_rn(__dsub_rn(yt, pos[3 * s + 1]), sy);
                    double dz = __dadd_rn(__dsub_rn(zt, pos[3 * s + 2]), sz);
                    double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
                    if (r < 1e-14) {
                        if (!origin) err = 2;
                        else if (s != t) err = err ? err : 1;
                        continue;
                    }
                    if (r < a.rc) img += q[s] * (erfc(a.xi * r) / r);
                }
                acc += img;
            }
    if (err) atomicMax(flag, err);
    double v = acc;
    if (a.add_self) v += (-2.0 * a.xi * q[t]) / a.sqrtpi;
    phi[t] = v;
}

static const int kRealUnit = 32;

// cells of edge >= rc/2 and the particle binning by cell
static void cell_bin(se_plan *pl, const double *pos, const double *q, int64_t N, RealArgs &a) {
    const double L = pl->L, rc = pl->p.rc;
    CellGeom &c = pl->cell;
    long long nn = (long long)std::floor(2.0 * L / rc);
    if (nn < 1) nn = 1;
    if (nn > 160) nn = 160;
    c.n = (int)nn;
    c.edge = L / c.n;
    for (int ax = 0; ax < 3; ++ax) c.mode[ax] = ax < pl->D ? (c.n >= 5 ? 1 : 2) : 0;
    a.n = c.n;
    a.edge = c.edge;
    for (int ax = 0; ax < 3; ++ax) a.mode[ax] = c.mode[ax];
    int nbins = c.n * c.n * c.n;
    cudaStream_t st = pl->stream;
    prof_begin(pl, SE_K_SORT);
    binning_reserve(pl->cbin, N, nbins, kRealUnit);
    SE_CUDA(cudaMemsetAsync(pl->cbin.counts.ptr, 0, sizeof(int) * (nbins + 1), st));
    cell_keys_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(pos, N, a, pl->cbin.keys.as<unsigned>(),
                                                                   pl->cbin.counts.as<int>());
    SE_LAUNCH_CHECK();
    pl->launches += 1;
    binning_sort(pl, pl->cbin, pos, q, N, nbins, kRealUnit);
    prof_end(pl, SE_K_SORT);
}

template <bool COUNT>
static void launch_cell(se_plan *pl, int64_t N, const RealArgs &a, double *phi, unsigned long long *npairs) {
    const CellGeom &c = pl->cell;
    int nbins = c.n * c.n * c.n;
    int64_t maxu = binning_max_units(pl->cbin, N, nbins, kRealUnit);
    bool mi = c.mode[0] == 2 || c.mode[1] == 2 || c.mode[2] == 2;
    unsigned blocks = (unsigned)((maxu + 3) / 4);
    cudaStream_t st = pl->stream;
    auto args = [&](auto kern) {
        kern<<<blocks, 128, 0, st>>>(pl->cbin.rec.as<double4>(), pl->cbin.idx_sorted.as<int>(),
                                     pl->cbin.starts.as<int>(), pl->cbin.units.as<int4>(), pl->cbin.nunits.as<int>(),
                                     a, phi, pl->flag.as<int>(), npairs);
    };
    if (!COUNT) prof_begin(pl, SE_K_REALSPACE);
    if (mi)
        args(realspace_cell_kernel<true, COUNT>);
    else
        args(realspace_cell_kernel<false, COUNT>);
    SE_LAUNCH_CHECK();
    if (!COUNT) prof_end(pl, SE_K_REALSPACE);
    pl->launches += 1;
}

void realspace_run(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi, int add_self, int rank,
                   int world) {
    const double L = pl->L, rc = pl->p.rc, xi = pl->p.xi;
    const int D = pl->D;
    if (!(xi > 0) || !(rc > 0)) fail(SE_EINVAL, "xi and rc must be positive");
    cudaStream_t st = pl->stream;
    pl->flag.ensure(sizeof(int) * 4);
    SE_CUDA(cudaMemsetAsync(pl->flag.ptr, 0, sizeof(int) * 4, st));
    if (world > 1) SE_CUDA(cudaMemsetAsync(phi, 0, sizeof(double) * (N > 0 ? N : 1), st));
    if (N <= 0) return;
    RealArgs a{};
    a.L = L;
    a.xi = xi;
    a.rc = rc;
    a.rc2 = rc * rc * (1.0 + 1e-12);  // prefilter only; the exact test is r < rc
    a.add_self = add_self;
    a.sqrtpi = std::sqrt(M_PI);
    a.rlo = N * rank / world;
    a.rhi = N * (rank + 1) / world;
    if (D >= 1 && rc > L / 2 + 1e-12) {
        int layers = (int)std::floor((rc + L / 2) / L) + 1;
        prof_begin(pl, SE_K_REALSPACE);
        realspace_image_kernel<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(pos, q, N, a.rlo, a.rhi, a, D, layers, phi,
                                                                           pl->flag.as<int>());
        SE_LAUNCH_CHECK();
        prof_end(pl, SE_K_REALSPACE);
        pl->launches += 1;
    } else {
        cell_bin(pl, pos, q, N, a);
        launch_cell<false>(pl, N, a, phi, nullptr);
    }
}

void realspace_pair_count(se_plan *pl, const double *pos, const double *q, int64_t N, long long *pairs) {
    const double L = pl->L, rc = pl->p.rc;
    if (pl->D >= 1 && rc > L / 2 + 1e-12) fail(SE_EINVAL, "pair counting covers the cell path (rc <= L/2)");
    *pairs = 0;
    if (N <= 0) return;
    RealArgs a{};
    a.L = L;
    a.xi = pl->p.xi;
    a.rc = rc;
    a.rc2 = rc * rc * (1.0 + 1e-12);
    a.sqrtpi = std::sqrt(M_PI);
    a.rlo = 0;
    a.rhi = N;
    pl->flag.ensure(sizeof(int) * 4);
    SE_CUDA(cudaMemsetAsync(pl->flag.ptr, 0, sizeof(int) * 4, pl->stream));
    pl->pairs.ensure(sizeof(unsigned long long));
    SE_CUDA(cudaMemsetAsync(pl->pairs.ptr, 0, sizeof(unsigned long long), pl->stream));
    cell_bin(pl, pos, q, N, a);
    launch_cell<true>(pl, N, a, nullptr, pl->pairs.as<unsigned long long>());
    unsigned long long h = 0;
    SE_CUDA(cudaMemcpyAsync(&h, pl->pairs.ptr, sizeof(h), cudaMemcpyDeviceToHost, pl->stream));
    SE_CUDA(cudaStreamSynchronize(pl->stream));
    *pairs = (long long)h;
}

}  // namespace se
