// Spreading (particle -> grid) and gathering (grid -> particle) for the SE
// Fourier pipeline: sekspace.spread / sekspace.gather (sekspace.py:105-178).
//
// Design (B200, fp64):
//  * Particles are binned by the TILE of their stencil start index
//    first = floor(u/h - P/2) + 1 (sekspace.py:114), stable-sorted, and split
//    into work units of <= UNIT particles (clustered inputs stay balanced).
//  * One CTA per unit accumulates into a zero-initialised padded tile of
//    (T+P-1)^3 doubles in shared memory.  fp64 shared-memory atomics are
//    CAS loops on sm_100a (ATOMS.CAST.SPIN.64), so the tile is updated with
//    plain LDS/DFMA/STS and made race free by ownership: warp w owns the
//    padded-tile x-planes lx == w (mod nwarps).  Every particle touches P
//    consecutive x-planes, so with nwarps | P each warp updates exactly
//    P/nwarps planes of every particle and no two warps ever touch the same
//    address.  Lanes cover the P*P (y,z) footprint; the (y,z) weight product
//    is formed once per particle and reused across the warp's planes.
//  * The window factors (3P per particle, fused Gaussian / ES / KB
//    evaluation) are computed once per particle into shared memory.
//  * The tile is flushed with native fp64 global reductions
//    (REDG.E.ADD.F64) into the L2-resident grid, wrapping periodic axes.
//  * Gather mirrors this: the padded tile of the grid is staged in shared
//    memory and a warp reduces each particle's P^3 stencil.
// Windows whose padded tile cannot fit in shared memory (P > ~24) use a
// direct kernel (one warp per particle, global fp64 reductions / loads).
#include "se_common.h"
#include "se_erfc_coeffs.h"

namespace se {

struct SpreadArgs {
    int P, M, Mt, D;
    int shape[3];
    double h, halfP;
    double off[3];
    int T, Tz, Tp, pitch, nwarps, batch;
    int nt[3];
    int lo[3];
    // window
    int window;
    double w, shapep, peak, mm, ww2, i0b;
    double invw, gcoef;  // 1/w and -m^2/(2 w^2)
    int64_t rlo, rhi;  // sorted-particle range of this shard
    double L;          // box edge (sane_coord)
};

// ---------------------------------------------------------------- windows
// exp(v) for v <= 0 by Cody-Waite reduction and the degree-11 polynomial of
// se_erfc_coeffs.h (coefficients as constant-bank operands; ~1 ulp).
__device__ __forceinline__ double exp_nonpos(double v) {
    if (v < -700.0) return 0.0;
    const double n = rint(v * SE_LOG2E);
    const double r = fma(n, -SE_LN2_LO, fma(n, -SE_LN2_HI, v));
    double e = se_exp_c[SE_EXP_NX];
#pragma unroll
    for (int i = SE_EXP_NX - 1; i >= 0; --i) e = fma(e, r, se_exp_c[i]);
    return e * __hiloint2double(((int)n + 1023) << 20, 0);
}

// windows.py:74-84 (Gaussian), 106-112 (KB), 148-154 (ES / BM); the
// divisions by w and 2w^2 are multiplications by host-computed reciprocals
// (<= 1 ulp from the reference's rounding).
template <int WIN>
__device__ __forceinline__ double window_eval(double x, const SpreadArgs &a) {
    if (!(fabs(x) <= a.w)) return 0.0;
    if (WIN == SE_WINDOW_GAUSSIAN) return a.peak * exp_nonpos(a.gcoef * (x * x));  // gcoef = -m^2 / (2 w^2)
    const double r = x * a.invw;
    double t = fma(-r, r, 1.0);
    t = t < 0.0 ? 0.0 : t;
    if (WIN == SE_WINDOW_BM) return exp_nonpos(a.shapep * (sqrt(t) - 1.0));
    return cyl_bessel_i0(a.shapep * sqrt(t)) / a.i0b;
}

// first stencil index along one axis (sekspace.py:113-114), IEEE division.
__device__ __forceinline__ long long stencil_first(double u, const SpreadArgs &a) {
    return (long long)floor(__dsub_rn(__ddiv_rn(u, a.h), a.halfP)) + 1;
}

__device__ __forceinline__ int start_index(long long first, int axis, const SpreadArgs &a) {
    if (axis < a.D) {
        // positions in [0, L) give first in [1 - P/2, M - P/2]: one wrap at
        // most (a 64-bit % is ~70 instructions); the exact path otherwise
        const int f = (int)first;
        int m = f < 0 ? f + a.M : (f >= a.M ? f - a.M : f);
        if ((long long)f != first || (unsigned)m >= (unsigned)a.M) {
            const long long mm = first % a.M;
            m = (int)(mm < 0 ? mm + a.M : mm);
        }
        return m;
    }
    return (int)first;
}

__device__ __forceinline__ int tile_coord(int s, int axis, const SpreadArgs &a) {
    int t = (s - a.lo[axis]) / (axis == 2 ? a.Tz : a.T);
    t = t < 0 ? 0 : t;
    return t >= a.nt[axis] ? a.nt[axis] - 1 : t;
}

__device__ __forceinline__ unsigned tile_key(const double *__restrict__ pos, int64_t i, const SpreadArgs &a) {
    int tc[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        double u = __dadd_rn(sane_coord(pos[3 * i + ax], a.L, i, ax), a.off[ax]);
        tc[ax] = tile_coord(start_index(stencil_first(u, a), ax, a), ax, a);
    }
    return (unsigned)((tc[0] * a.nt[1] + tc[1]) * a.nt[2] + tc[2]);
}

__global__ void tile_keys_kernel(const double *__restrict__ pos, int64_t N, SpreadArgs a,
                                 unsigned *__restrict__ keys, int *__restrict__ counts) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const unsigned key = tile_key(pos, i, a);
    keys[i] = key;
    atomicAdd(&counts[key], 1);
}

// Few tiles (<= kTileHistSmem): per-block shared-memory histogram flushed
// once per non-empty tile (hundreds of particles per tile contend on one
// global counter otherwise: 44 -> ~15 us at cfg2).
constexpr int kTileHistSmem = 8192;
__global__ void tile_keys_hist_kernel(const double *__restrict__ pos, int64_t N, SpreadArgs a, int nbins,
                                      unsigned *__restrict__ keys, int *__restrict__ counts) {
    extern __shared__ int hist[];
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned key = tile_key(pos, i, a);
        keys[i] = key;
        atomicAdd(&hist[key], 1);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nbins; b += blockDim.x)
        if (hist[b]) atomicAdd(&counts[b], hist[b]);
}

// Window-factor layout (stage_batch): factor t of (particle p, axis) at
// wts[(3 p + axis) EA + t ET].  P = 8 (compile time): EA = 1, ET = 3 batch
// + 1, i.e. [t][p][axis] -- measured 0.59 -> 0.53 ms spread, 0.36 -> 0.33 ms
// gather at cfg2; other P keep [p][axis][t] (EA = P, ET = 1: the
// transposed layout measured slower at P = 10).
constexpr bool wts_transposed(int PC) { return PC == 8; }
__host__ __device__ constexpr int tile_batch(int P) { return P >= 12 ? 32 : 64; }
__host__ __device__ constexpr int wts_ea(int PC, int P) { return wts_transposed(PC) ? 1 : P; }
__host__ __device__ constexpr int wts_et(int PC, int batch) { return wts_transposed(PC) ? 3 * batch + 1 : 1; }

// Stage the 3P window factors of a batch of particles.  wts layout: see
// wts_ea / wts_et (transposed for P = 8: a task (p, axis) writes its P
// factors 3 batch + 1 doubles apart, so consecutive tasks hit consecutive
// banks -- the [p][axis][t] layout makes every staging store 8-way
// conflicted; the odd stride keeps the consumers' reads conflict free);
// loc: [p][4] = the local start (x, y, z) within the padded tile as bytes
// 0..2 of loc[p][0] (one broadcast LDS.32 for the consumers instead of
// three; each axis task writes its own byte), loc[p][3] = the caller-order
// index sidx[s] (gather; loaded here, off the store's critical path) or the
// sorted index (sidx == nullptr).  FOLDQ multiplies the x factors by the
// charge.  PC > 0 is the window support P as a compile-time constant (0:
// runtime a.P).
template <int WIN, bool FOLDQ, int PC>
__device__ __forceinline__ void stage_batch(const double4 *__restrict__ rec, int s0, int nb, const int org[3],
                                            const SpreadArgs &a, double *wts, int *loc,
                                            const int *__restrict__ sidx = nullptr, int tid = -1, int nthr = 0) {
    const int P = PC > 0 ? PC : a.P;
    if (tid < 0) {
        tid = threadIdx.x;
        nthr = blockDim.x;
    }
    for (int task = tid; task < nb * 3; task += nthr) {
        int p = task / 3, ax = task - 3 * p;
        double4 r = rec[s0 + p];
        double x = ax == 0 ? r.x : (ax == 1 ? r.y : r.z);
        double u = __dadd_rn(x, a.off[ax]);
        long long f = stencil_first(u, a);
        // factor t of (p, axis) at wts[(3 p + axis) EA + t ET] (wts_strides)
        const int EA = wts_ea(PC, P), ET = wts_et(PC, PC > 0 ? tile_batch(PC) : a.batch);
        double *wo = wts + (p * 3 + ax) * EA;
#pragma unroll
        for (int t = 0; t < (PC > 0 ? PC : 64); ++t) {
            if (PC == 0 && t >= P) break;
            double d = __dsub_rn(__dmul_rn((double)(f + t), a.h), u);  // sekspace.py:116
            double v = window_eval<WIN>(d, a);
            if (FOLDQ && ax == 0) v = __dmul_rn(r.w, v);
            wo[t * ET] = v;
        }
        reinterpret_cast<unsigned char *>(loc + p * 4)[ax] = (unsigned char)(start_index(f, ax, a) - org[ax]);
        if (ax == 0) loc[p * 4 + 3] = sidx ? sidx[s0 + p] : s0 + p;
    }
}

__device__ __forceinline__ void unit_origin(int bin, const SpreadArgs &a, int org[3]) {
    int tz = bin % a.nt[2];
    int ty = (bin / a.nt[2]) % a.nt[1];
    int tx = bin / (a.nt[2] * a.nt[1]);
    org[0] = a.lo[0] + tx * a.T;
    org[1] = a.lo[1] + ty * a.T;
    org[2] = a.lo[2] + tz * a.Tz;
}

// Per-axis grid index of every padded-tile coordinate (-1 off the grid),
// wrapped on periodic axes: gmap[ax * Tp + l] (x, y: Tp entries; z: pitch).
#ifndef TILE_FLAT
#define TILE_FLAT 1
#endif
template <int PC>
struct TileC;
__device__ __forceinline__ void build_axis_maps(const int org[3], const SpreadArgs &a, int *gmap) {
    for (int i = threadIdx.x; i < 2 * a.Tp + a.pitch; i += blockDim.x) {
        const int ax = min(i / a.Tp, 2), l = i - ax * a.Tp;
        int g = org[ax] + l;
        if (ax < a.D)
            g %= a.M;
        else if (g < 0 || g >= a.Mt)
            g = -1;
        gmap[i] = g;
    }
}

// Visit every padded-tile cell with its grid index: one warp per (lx, ly)
// row, lanes along z (coalesced in the grid's z-fastest layout).
template <int PC = 0, class F>
__device__ __forceinline__ void for_tile_cells(const SpreadArgs &a, const int *gmap, F f) {
    if constexpr (PC > 0 && TILE_FLAT && TileC<PC>::T > 0) {
        // compile-time tile geometry: the cells as one flat range over all
        // threads (every lane busy; the row / column split is a multiply by a
        // constant instead of a runtime division)
        constexpr int Tp = TileC<PC>::Tp, pitch = TileC<PC>::pitch, ncell = Tp * Tp * pitch;
        const long long s1 = a.shape[1], s2 = a.shape[2];
        for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
            const int row = i / pitch, lz = i - row * pitch;
            const int lx = row / Tp, ly = row - lx * Tp;
            const int gx = gmap[lx], gy = gmap[Tp + ly], gz = gmap[2 * Tp + lz];
            f(i, (gx | gy | gz) >= 0 ? ((long long)gx * s1 + gy) * s2 + gz : -1LL);
        }
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const int Tp = a.Tp;
    for (int row = warp; row < Tp * Tp; row += nwarp) {
        const int lx = row / Tp, ly = row - lx * Tp;
        const int gx = gmap[lx], gy = gmap[Tp + ly];
        const bool rok = gx >= 0 && gy >= 0;
        const long long gbase = ((long long)gx * a.shape[1] + gy) * a.shape[2];
        const int tbase = (lx * Tp + ly) * a.pitch;
        for (int lz = lane; lz < a.pitch; lz += 32) {
            const int gz = gmap[2 * Tp + lz];
            f(tbase + lz, rok && gz >= 0 ? gbase + gz : -1LL);
        }
    }
}

// Per-lane share of the P x P (y, z) footprint: lane handles pairs
// pi = lane + 32 it; with compile-time P the pair coordinates are computed
// once per CTA instead of per particle.
// Tile geometry as a function of P alone (tile_setup's rule), so that the
// compile-time-P kernels also know Tp, pitch and plane at compile time: the
// stencil loads then use immediate offsets instead of per-load address math.
//
// Bank-conflict-free stencil rows: lane l of a warp handles (y, z) pair
// pi = l + 32 it of the P x P footprint at word offset ty * pitch + tz; with
// pitch == P (mod 16) that offset is == pi (mod 16), so the 32 lanes hit
// every bank pair exactly twice (the minimum for 8-byte words).  The padded
// z extent is therefore Tz + P - 1 with Tz == 1 (mod 16): tiles are
// T x T x 17 for P <= 12, the padding doing useful work instead of being
// wasted columns.  Wider windows keep cubic tiles (a 17-deep tile would
// leave only a sliver in x and y) with the old padded pitch: rows of 16
// (P = 16) are conflict free as they are, P == 8 (mod 16) pads to == 8.
// The budget keeps 3 CTAs per SM (228 KB, 1 KB reserved per CTA): measured
// at P = 8, 3 CTAs per SM beat both 2 (larger tiles) and 4 (smaller tiles).
constexpr size_t kSmemSM = 228 * 1024, kSmemReserved = 1024;
constexpr size_t kSmemFirst = kSmemSM / 3 - kSmemReserved;
constexpr bool tile_aniso(int P) { return P % 16 != 0 && P <= 12; }
constexpr int tile_Tz(int T, int P) { return tile_aniso(P) ? 17 : T; }
constexpr int tile_pitch(int T, int P) {
    return tile_aniso(P) ? 17 + P - 1
                         : (P % 16 == 8 ? T + P - 1 + ((8 - (T + P - 1) % 16) + 16) % 16 : T + P - 1);
}
constexpr size_t tile_bytes(int T, int P) {
    return sizeof(double) * ((size_t)(T + P - 1) * (T + P - 1) * tile_pitch(T, P) +
                             (size_t)(tile_batch(P) * 3 + (wts_transposed(P) ? 1 : 0)) * P) +
           sizeof(int) * (4 * tile_batch(P) + 2 * (T + P - 1) + tile_pitch(T, P));
}
// P = 8: 8 x 8 x 17 tiles measured 0.5% faster per cfg2 step than 10 x 10 x 17
#ifndef SE_TILE_TMAX8
#define SE_TILE_TMAX8 8
#endif
constexpr int tile_Tmax(int P) { return P == 8 ? SE_TILE_TMAX8 : 16; }
constexpr int tile_T(int P) {
    constexpr int cand[] = {16, 14, 12, 10, 8, 6, 4, 2, 1};
    for (int T : cand)
        if (T <= tile_Tmax(P) && tile_bytes(T, P) <= kSmemFirst) return T;
    return 0;
}
template <int PC>
struct TileC {
    static constexpr int T = PC > 0 ? tile_T(PC) : 0;
    static constexpr int Tp = T > 0 ? T + PC - 1 : 0;
    static constexpr int pitch = T > 0 ? tile_pitch(T, PC) : 0;
    static constexpr int plane = Tp * pitch;
};

// Lanes per row of pairs: pi = lane + LW it.  With LW a multiple of P a
// lane's z offset tz = pi mod P is the same in every iteration, so its z
// factor is loaded ONCE per particle (one shared-memory wavefront per
// iteration less): P = 8, 16 have LW = 32 anyway; P = 10 uses 30 lanes (4
// iterations of 30, 30, 30, 10 pairs instead of 32, 32, 32, 4: the same
// number of tile wavefronts, 5 factor loads instead of 8).  For lanes < LW
// the bank pattern is the one described above (offset == pi mod 16).
#ifndef SE_LANEPAIR_TZ
#define SE_LANEPAIR_TZ 1
#endif
// The (y, z) products before the plane's read-modify-writes (all factor
// loads issued first): P = 8 (round 2, first session), and with the single
// z-factor load also P = 10, 12 (-3% / -2.5% spread; P = 16: +5%, not used).
#ifndef SE_YZ_FIRST_MAXP
#define SE_YZ_FIRST_MAXP 12
#endif
constexpr bool yz_first(int PC) { return wts_transposed(PC) || (PC > 0 && PC <= SE_YZ_FIRST_MAXP); }
constexpr int lanepair_width(int PC, bool narrow) { return (SE_LANEPAIR_TZ && narrow && PC == 10) ? 30 : 32; }
// NARROW: the spreading kernels (measured at P = 10: spread -9%, the gather
// +12..20% -- it keeps 32 lanes).
template <int PC, bool NARROW = true>
struct LanePairs {
    static constexpr int LW = lanepair_width(PC, NARROW);
    static constexpr int NPI = PC > 0 ? (PC * PC + LW - 1) / LW : 1;
    // every iteration of a lane has the same tz
    static constexpr bool TZC = SE_LANEPAIR_TZ && PC > 0 && LW % (PC > 0 ? PC : 1) == 0;
    int ty[NPI], tz[NPI], off[NPI];
    __device__ __forceinline__ void init(int lane, int pitch) {
#pragma unroll
        for (int it = 0; it < NPI; ++it) {
            const int pi = lane + LW * it;
            ty[it] = pi / (PC > 0 ? PC : 1);
            tz[it] = pi - ty[it] * (PC > 0 ? PC : 1);
            off[it] = ty[it] * pitch + tz[it];
        }
    }
    __device__ __forceinline__ bool valid(int lane, int it) const { return lane < LW && lane + LW * it < PC * PC; }
};

template <int WIN, int PC>
__global__ void __launch_bounds__(512) spread_tile_kernel(const double4 *__restrict__ rec, const int4 *__restrict__ units,
                                                          const int *__restrict__ nunits, SpreadArgs a,
                                                          double *__restrict__ grid, double *__restrict__ dbuf) {
    if ((int)blockIdx.x >= *nunits) return;
    int4 un = units[blockIdx.x];
    int ubeg = (int)max((int64_t)un.y, a.rlo), uend = (int)min((int64_t)un.y + un.z, a.rhi);
    if (ubeg >= uend) return;
    extern __shared__ double smem[];
    // compile-time geometry for compile-time P (tile_setup checks it matches)
    const int P = PC > 0 ? PC : a.P, Tp = TileC<PC>::T > 0 ? TileC<PC>::Tp : a.Tp,
              pitch = TileC<PC>::T > 0 ? TileC<PC>::pitch : a.pitch, plane = Tp * pitch;
    const int ncell = Tp * plane;
    double *tile = smem;
    double *wts = tile + ncell;
    const int BATCH = PC > 0 ? tile_batch(PC) : a.batch;  // a.batch == tile_batch(P) (tile_setup)
    int *loc = reinterpret_cast<int *>(wts + (BATCH * 3 + (wts_transposed(PC) ? 1 : 0)) * P);
    const int EA = wts_ea(PC, P), S = wts_et(PC, BATCH);  // wts strides (stage_batch)
    int *gmap = loc + 4 * BATCH;
    int org[3];
    unit_origin(un.x, a, org);
    for (int i = threadIdx.x; i < ncell; i += blockDim.x) tile[i] = 0.0;
    build_axis_maps(org, a, gmap);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = a.nwarps;
    const int npair = P * P;
    LanePairs<PC> lp;
    lp.init(lane, pitch);
    for (int b0 = ubeg; b0 < uend; b0 += BATCH) {
        int nb = min(BATCH, uend - b0);
        __syncthreads();  // tile zeroed / previous batch consumed
        stage_batch<WIN, true, PC>(rec, b0, nb, org, a, wts, loc);
        __syncthreads();
        for (int p = 0; p < nb; ++p) {
            const int pk = loc[p * 4];
            const int lx0 = pk & 0xff, ly0 = (pk >> 8) & 0xff, lz0 = (pk >> 16) & 0xff;
            const double *wx = wts + p * 3 * EA, *wy = wx + EA, *wz = wx + 2 * EA;  // factor t at [t * S]
            if (PC > 0) {
                // nwarps == P: this warp owns exactly one x-plane of the
                // particle; at P = 8 the (y, z) products are formed before
                // the plane's read-modify-writes (all weight loads issued
                // first: 0.60 -> 0.55 ms at cfg2; slower at P = 10)
                int t0 = (warp - lx0) % PC;
                t0 = t0 < 0 ? t0 + PC : t0;
                const double wxt = wx[t0 * S];
                double *base = tile + (lx0 + t0) * plane + ly0 * pitch + lz0;
                // z factor: one load per particle when tz does not depend on it
                const double wzc = LanePairs<PC>::TZC ? wz[lp.tz[0] * S] : 0.0;
                if (yz_first(PC)) {
                    double yz[LanePairs<PC>::NPI];
#pragma unroll
                    for (int it = 0; it < LanePairs<PC>::NPI; ++it)
                        yz[it] = lp.valid(lane, it)
                                     ? __dmul_rn(wy[lp.ty[it] * S], LanePairs<PC>::TZC ? wzc : wz[lp.tz[it] * S])
                                     : 0.0;
#pragma unroll
                    for (int it = 0; it < LanePairs<PC>::NPI; ++it) {
                        if (lp.valid(lane, it)) {
                            double *c = base + lp.off[it];
                            *c = fma(wxt, yz[it], *c);
                        }
                    }
                } else {
#pragma unroll
                    for (int it = 0; it < LanePairs<PC>::NPI; ++it) {
                        if (lp.valid(lane, it)) {
                            double *c = base + lp.off[it];
                            *c = fma(wxt, __dmul_rn(wy[lp.ty[it] * S], LanePairs<PC>::TZC ? wzc : wz[lp.tz[it] * S]),
                                     *c);
                        }
                    }
                }
            } else {
                int t0 = (warp - lx0) % nw;
                t0 = t0 < 0 ? t0 + nw : t0;
                for (int pi = lane; pi < npair; pi += 32) {
                    int ty = pi / P, tz = pi - ty * P;
                    double cyz = __dmul_rn(wy[ty * S], wz[tz * S]);
                    int off = (ly0 + ty) * pitch + lz0 + tz;
                    for (int t = t0; t < P; t += nw) {
                        double *c = tile + (lx0 + t) * plane + off;
                        *c = fma(wx[t * S], cyz, *c);
                    }
                }
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (dbuf) {
        // deterministic mode: the unit's padded tile as it is (coalesced
        // stores); spread_det_reduce_kernel sums the units in a fixed order
        double *o = dbuf + (size_t)blockIdx.x * ncell;
        for (int i = threadIdx.x; i < ncell; i += blockDim.x) o[i] = tile[i];
        return;
    }
    for_tile_cells<PC>(a, gmap, [&](int ti, long long gi) {
        const double v = tile[ti];
        if (gi >= 0 && v != 0.0) atomicAdd(grid + gi, v);
    });
}

// Deterministic spreading, second pass: every grid point sums the cells of
// the per-unit padded tiles that map onto it -- candidate tiles in
// ascending (x, y, z) tile order, a tile's units in order -- so the grid is
// bitwise reproducible (the atomic tile flush adds in arbitrary order).
__global__ void spread_det_reduce_kernel(const double *__restrict__ dbuf, const int4 *__restrict__ units,
                                         const int *__restrict__ ubstart, SpreadArgs a, int64_t G,
                                         double *__restrict__ grid) {
    const int ext[3] = {a.Tp, a.Tp, a.pitch};
    const int te[3] = {a.T, a.T, a.Tz};
    const int plane = a.Tp * a.pitch, ncell = a.Tp * plane;
    // first local coordinate of grid index g in the padded tile t along
    // axis ax (-1: not covered); on a periodic axis the padded tile may wrap
    // onto g more than once (l, l + M, ... < ext: a tile wider than the grid)
    // and a wide window with small tiles has up to ceil((T + P - 1) / T)
    // covering tiles per axis
    auto local = [&](int ax, int g, int t) {
        int l = g - (a.lo[ax] + t * te[ax]);
        if (ax < a.D) l = ((l % a.M) + a.M) % a.M;
        return (l >= 0 && l < ext[ax]) ? l : -1;
    };
    auto step = [&](int ax) { return ax < a.D ? a.M : 1 << 30; };
    for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < G; gi += (int64_t)gridDim.x * blockDim.x) {
        const int gz = (int)(gi % a.shape[2]);
        const int gy = (int)((gi / a.shape[2]) % a.shape[1]);
        const int gx = (int)(gi / ((int64_t)a.shape[2] * a.shape[1]));
        double v = 0.0;
        for (int tx = 0; tx < a.nt[0]; ++tx)
            for (int lx = local(0, gx, tx); lx >= 0 && lx < ext[0]; lx += step(0))
                for (int ty = 0; ty < a.nt[1]; ++ty)
                    for (int ly = local(1, gy, ty); ly >= 0 && ly < ext[1]; ly += step(1))
                        for (int tz = 0; tz < a.nt[2]; ++tz)
                            for (int lz = local(2, gz, tz); lz >= 0 && lz < ext[2]; lz += step(2)) {
                                const int b = (tx * a.nt[1] + ty) * a.nt[2] + tz;
                                const int off = lx * plane + ly * a.pitch + lz;
                                for (int u = ubstart[b]; u < ubstart[b + 1]; ++u) {
                                    const int4 un = units[u];
                                    if ((int64_t)un.y + un.z <= a.rlo || (int64_t)un.y >= a.rhi) continue;
                                    v += dbuf[(size_t)u * ncell + off];
                                }
                            }
        grid[gi] = v;
    }
}

// Warp-specialised spreading (P = 8): kSwsC plane-owner warps update the
// tile with a staged batch while kSwsP producer warps stage the next batch
// into the other of two factor / record buffers, handed over by named
// barriers (FULL[b]: producers arrive, owners wait; EMPTY[b]: owners
// arrive, producers wait) -- the CTA-wide barriers around each batch's
// staging in spread_tile_kernel are gone.  SE_B200_SPREAD_WS=0: the
// single-role kernel.
constexpr int kSwsC = 8, kSwsP = 4;
constexpr int kBarFull0 = 1, kBarEmpty0 = 3;  // ids 1, 2 and 3, 4 (0: __syncthreads)
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr size_t spread_ws_extra(int P) {  // the second factor + record buffer
    return sizeof(double) * (size_t)(tile_batch(P) * 3 + 1) * P + sizeof(int) * 4 * tile_batch(P);
}

template <int WIN>
__global__ void __launch_bounds__(32 * (kSwsC + kSwsP), 3) spread_ws_kernel(const double4 *__restrict__ rec,
                                                                             const int4 *__restrict__ units,
                                                                             const int *__restrict__ nunits,
                                                                             SpreadArgs a, double *__restrict__ grid) {
    constexpr int PC = 8, B = tile_batch(PC), NT = 32 * (kSwsC + kSwsP);
    static_assert(wts_transposed(PC), "the warp-specialised spread uses the transposed factor layout");
    if ((int)blockIdx.x >= *nunits) return;
    const int4 un = units[blockIdx.x];
    const int ubeg = (int)max((int64_t)un.y, a.rlo), uend = (int)min((int64_t)un.y + un.z, a.rhi);
    if (ubeg >= uend) return;
    extern __shared__ double smem[];
    constexpr int Tp = TileC<PC>::Tp, pitch = TileC<PC>::pitch, plane = Tp * pitch, ncell = Tp * plane;
    constexpr int WSZ = (B * 3 + 1) * PC, S = wts_et(PC, B);
    double *tile = smem;
    double *const wts0 = tile + ncell;                                 // buffer b: wts0 + b WSZ
    int *const loc0 = reinterpret_cast<int *>(tile + ncell + 2 * WSZ);  // buffer b: loc0 + 4 b B
    int *gmap = loc0 + 8 * B;
    int org[3];
    unit_origin(un.x, a, org);
    for (int i = threadIdx.x; i < ncell; i += blockDim.x) tile[i] = 0.0;
    build_axis_maps(org, a, gmap);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nbatch = (uend - ubeg + B - 1) / B;
    if (warp >= kSwsC) {
        // producers
        const int tid = threadIdx.x - 32 * kSwsC;
        for (int k = 0; k < nbatch; ++k) {
            const int b = k & 1, b0 = ubeg + k * B, nb = min(B, uend - b0);
            if (k >= 2) named_sync(kBarEmpty0 + b, NT);
            stage_batch<WIN, true, PC>(rec, b0, nb, org, a, wts0 + b * WSZ, loc0 + 4 * b * B, nullptr, tid,
                                       32 * kSwsP);
            __threadfence_block();
            named_arrive(kBarFull0 + b, NT);
        }
    } else {
        // plane owners: warp w owns the padded tile's x planes lx == w (mod 8)
        LanePairs<PC> lp;
        lp.init(lane, pitch);
        for (int k = 0; k < nbatch; ++k) {
            const int b = k & 1, b0 = ubeg + k * B, nb = min(B, uend - b0);
            named_sync(kBarFull0 + b, NT);
            const double *wts = wts0 + b * WSZ;
            const int *loc = loc0 + 4 * b * B;
            for (int p = 0; p < nb; ++p) {
                const int pk = loc[p * 4];
                const int lx0 = pk & 0xff, ly0 = (pk >> 8) & 0xff, lz0 = (pk >> 16) & 0xff;
                const double *wx = wts + p * 3, *wy = wx + 1, *wz = wx + 2;  // factor t at [t * S]
                int t0 = (warp - lx0) % PC;
                t0 = t0 < 0 ? t0 + PC : t0;
                const double wxt = wx[t0 * S];
                double *base = tile + (lx0 + t0) * plane + ly0 * pitch + lz0;
                double yz[LanePairs<PC>::NPI];
                const double wzc = LanePairs<PC>::TZC ? wz[lp.tz[0] * S] : 0.0;  // tz is the same in both iterations
#pragma unroll
                for (int it = 0; it < LanePairs<PC>::NPI; ++it)
                    yz[it] = __dmul_rn(wy[lp.ty[it] * S], LanePairs<PC>::TZC ? wzc : wz[lp.tz[it] * S]);
#pragma unroll
                for (int it = 0; it < LanePairs<PC>::NPI; ++it) {
                    double *c = base + lp.off[it];
                    *c = fma(wxt, yz[it], *c);
                }
                __syncwarp();
            }
            if (k + 2 < nbatch) named_arrive(kBarEmpty0 + b, NT);
        }
    }
    __syncthreads();
    for_tile_cells<PC>(a, gmap, [&](int ti, long long gi) {
        const double v = tile[ti];
        if (gi >= 0 && v != 0.0) atomicAdd(grid + gi, v);
    });
}

template <int WIN, int PC>
// P >= 10 (384+ threads): cap registers at 64 so that two CTAs fit per SM
// (86 registers left a single 12-warp CTA per SM at P = 12)
__global__ void __launch_bounds__(512, (PC >= 10 ? 2 : 0)) gather_tile_kernel(const double4 *__restrict__ rec, const int *__restrict__ sidx,
                                                          const int4 *__restrict__ units, const int *__restrict__ nunits,
                                                          SpreadArgs a, const double *__restrict__ grid,
                                                          double *__restrict__ phi, double h3, int accumulate) {
    if ((int)blockIdx.x >= *nunits) return;
    int4 un = units[blockIdx.x];
    int ubeg = (int)max((int64_t)un.y, a.rlo), uend = (int)min((int64_t)un.y + un.z, a.rhi);
    if (ubeg >= uend) return;
    extern __shared__ double smem[];
    // compile-time geometry for compile-time P (tile_setup checks it matches)
    const int P = PC > 0 ? PC : a.P, Tp = TileC<PC>::T > 0 ? TileC<PC>::Tp : a.Tp,
              pitch = TileC<PC>::T > 0 ? TileC<PC>::pitch : a.pitch, plane = Tp * pitch;
    const int ncell = Tp * plane;
    double *tile = smem;
    double *wts = tile + ncell;
    const int BATCH = PC > 0 ? tile_batch(PC) : a.batch;  // a.batch == tile_batch(P) (tile_setup)
    int *loc = reinterpret_cast<int *>(wts + (BATCH * 3 + (wts_transposed(PC) ? 1 : 0)) * P);
    const int EA = wts_ea(PC, P), S = wts_et(PC, BATCH);  // wts strides (stage_batch)
    int *gmap = loc + 4 * BATCH;
    int org[3];
    unit_origin(un.x, a, org);
    build_axis_maps(org, a, gmap);
    __syncthreads();
    // the padded tile by asynchronous 8-byte copies (cp.async, LDGSTS): a
    // thread issues all its cells' loads back to back instead of waiting
    // for each one in a register round trip
    for_tile_cells<PC>(a, gmap, [&](int ti, long long gi) {
        if (gi >= 0)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(tile + ti)),
                         "l"(grid + gi));
        else
            tile[ti] = 0.0;
    });
    asm volatile("cp.async.wait_all;" ::: "memory");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = a.nwarps;
    const int npair = P * P;
    LanePairs<PC, false> lp;
    lp.init(lane, pitch);
    for (int b0 = ubeg; b0 < uend; b0 += BATCH) {
        int nb = min(BATCH, uend - b0);
        __syncthreads();
        // P = 8: the caller-order index is loaded at staging (off the
        // store's critical path; slower at P = 10), else at the store
        stage_batch<WIN, false, PC>(rec, b0, nb, org, a, wts, loc, wts_transposed(PC) ? sidx : nullptr);
        __syncthreads();
        // this lane's share of particle p's P^3 sum
        auto partial = [&](int p) -> double {
            const int pk = loc[p * 4];
            const int lx0 = pk & 0xff, ly0 = (pk >> 8) & 0xff, lz0 = (pk >> 16) & 0xff;
            const double *wx = wts + p * 3 * EA, *wy = wx + EA, *wz = wx + 2 * EA;  // factor t at [t * S]
            double acc = 0.0;
            if (PC > 0) {
                const double *base = tile + lx0 * plane + ly0 * pitch + lz0;
                const double wzc = LanePairs<PC, false>::TZC ? wz[lp.tz[0] * S] : 0.0;
#pragma unroll
                for (int it = 0; it < LanePairs<PC, false>::NPI; ++it) {
                    if (lp.valid(lane, it)) {
                        const double *c = base + lp.off[it];
                        double s = 0.0;
#pragma unroll
                        for (int t = 0; t < PC; ++t) s = fma(wx[t * S], c[t * plane], s);
                        acc = fma(__dmul_rn(wy[lp.ty[it] * S], LanePairs<PC, false>::TZC ? wzc : wz[lp.tz[it] * S]), s, acc);
                    }
                }
            } else {
                for (int pi = lane; pi < npair; pi += 32) {
                    int ty = pi / P, tz = pi - ty * P;
                    const double *c = tile + lx0 * plane + (ly0 + ty) * pitch + lz0 + tz;
                    double s = 0.0;
                    for (int t = 0; t < P; ++t) s = fma(wx[t * S], c[t * plane], s);
                    acc = fma(__dmul_rn(wy[ty * S], wz[tz * S]), s, acc);
                }
            }
            return acc;
        };
        auto store = [&](int p, double acc) {
            const int orig = wts_transposed(PC) ? loc[p * 4 + 3] : sidx[loc[p * 4 + 3]];
            const double v = acc * h3;
            phi[orig] = accumulate ? phi[orig] + v : v;
        };
        // two particles per pass with one reduce-scatter: after the xor-16
        // exchange lanes 0-15 hold particle p's pair sums, lanes 16-31 those
        // of p + nw (5 shuffles for two particles instead of 10)
        int p = warp;
        for (; p + nw < nb; p += 2 * nw) {
            const double a0 = partial(p), a1 = partial(p + nw);
            const bool hi = (lane & 16) != 0;
            double v = hi ? a1 : a0;
            v += __shfl_xor_sync(0xffffffffu, hi ? a0 : a1, 16);
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((lane & 15) == 0) store(hi ? p + nw : p, v);
        }
        if (p < nb) {
            double acc = partial(p);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) store(p, acc);
        }
    }
}

// ---------------------------------------------------- large-P direct path
template <int WIN, bool SPREAD>
__global__ void direct_kernel(const double4 *__restrict__ rec, const int *__restrict__ sidx, int64_t rlo, int64_t rhi,
                              SpreadArgs a, double *__restrict__ grid, const double *__restrict__ gin,
                              double *__restrict__ phi, double h3, int accumulate) {
    extern __shared__ double smem[];
    const int P = a.P;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *w = smem + warp * 3 * P;
    int64_t i = rlo + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (i >= rhi) return;
    double4 r = rec[i];
    long long f[3];
    int s[3];
    for (int ax = 0; ax < 3; ++ax) {
        double x = ax == 0 ? r.x : (ax == 1 ? r.y : r.z);
        double u = __dadd_rn(x, a.off[ax]);
        f[ax] = stencil_first(u, a);
        s[ax] = start_index(f[ax], ax, a);
        for (int t = lane; t < P; t += 32) {
            double d = __dsub_rn(__dmul_rn((double)(f[ax] + t), a.h), u);
            double v = window_eval<WIN>(d, a);
            if (SPREAD && ax == 0) v = __dmul_rn(r.w, v);
            w[ax * P + t] = v;
        }
    }
    __syncwarp();
    double acc = 0.0;
    for (int pi = lane; pi < P * P; pi += 32) {
        int ty = pi / P, tz = pi - ty * P;
        int gy = s[1] + ty, gz = s[2] + tz;
        if (1 < a.D) gy %= a.M;
        if (2 < a.D) gz %= a.M;
        if (gy >= a.shape[1] || gz >= a.shape[2]) continue;
        double cyz = __dmul_rn(w[P + ty], w[2 * P + tz]);
        double sacc = 0.0;
        for (int t = 0; t < P; ++t) {
            int gx = s[0] + t;
            if (0 < a.D) gx %= a.M;
            if (gx >= a.shape[0]) continue;
            long long gi = ((long long)gx * a.shape[1] + gy) * a.shape[2] + gz;
            if (SPREAD)
                atomicAdd(grid + gi, w[t] * cyz);
            else
                sacc = fma(w[t], gin[gi], sacc);
        }
        if (!SPREAD) acc = fma(cyz, sacc, acc);
    }
    if (!SPREAD) {
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            int orig = sidx[i];
            double v = acc * h3;
            phi[orig] = accumulate ? phi[orig] + v : v;
        }
    }
}

// --------------------------------------------------------------- host side
static SpreadArgs make_args(se_plan *pl) {
    const se_grid_t &g = pl->g;
    const se_params_t &p = pl->p;
    SpreadArgs a{};
    a.P = p.P;
    a.M = g.M;
    a.Mt = g.Mt;
    a.D = g.D;
    for (int i = 0; i < 3; ++i) {
        a.shape[i] = g.shape[i];
        a.off[i] = g.offsets[i];
    }
    a.h = g.h;
    a.L = pl->L;
    a.halfP = 0.5 * p.P;
    a.window = p.window;
    a.w = 0.5 * p.P * g.h;
    a.shapep = p.shape;
    a.peak = p.shape / (a.w * std::sqrt(2.0 * M_PI));
    a.mm = p.shape * p.shape;
    a.ww2 = 2.0 * a.w * a.w;
    a.invw = 1.0 / a.w;
    a.gcoef = -a.mm / a.ww2;
    a.i0b = 1.0;
    if (p.window == SE_WINDOW_KB) a.i0b = bessel_i0(p.shape);
    const TileGeom &t = pl->tile;
    a.T = t.T;
    a.Tz = t.Tz;
    a.Tp = t.Tp;
    a.pitch = t.pitch;
    a.nwarps = t.nwarps;
    a.batch = t.batch;
    for (int i = 0; i < 3; ++i) {
        a.nt[i] = t.nt[i];
        a.lo[i] = t.lo[i];
    }
    return a;
}

static const int kUnit = 1024;     // particles per spreading work unit
static const size_t kSmemCap = 200 * 1024;
// preferred per-CTA budget: 4 CTAs per SM (the per-particle loop is latency
// bound, so occupancy beats the smaller halo of larger tiles)

void tile_setup(se_plan *pl) {
    TileGeom &t = pl->tile;
    if (t.T) return;
    const int P = pl->p.P;
    int nw = P <= 16 ? P : 16;
    while (nw > 1 && P % nw) --nw;
    if (nw < 4 && P > 4) nw = P < 16 ? P : 16;  // keep enough warps even if nw does not divide P
    t.nwarps = nw;
    t.batch = tile_batch(P);
    const int cand[] = {16, 14, 12, 10, 8, 6, 4, 2, 1};
    t.T = 0;
    for (size_t pass = 0; pass < 2 && !t.T; ++pass) {
        size_t cap = pass == 0 ? kSmemFirst : kSmemCap;
        for (int T : cand) {
            const size_t bytes = tile_bytes(T, P);  // the same rule as TileC (compile-time P)
            if (T <= tile_Tmax(P) && bytes <= cap) {
                t.T = T;
                t.Tz = tile_Tz(T, P);
                t.Tp = T + P - 1;
                t.pitch = tile_pitch(T, P);
                t.smem = bytes;
                break;
            }
        }
    }
    if (!t.T) {  // direct path
        t.T = -1;
        t.Tz = -1;
        t.Tp = 0;
        t.pitch = 0;
        t.smem = 0;
        for (int i = 0; i < 3; ++i) {
            t.nt[i] = 1;
            t.lo[i] = 0;
        }
        return;
    }
    for (int ax = 0; ax < 3; ++ax) {
        int extent = ax < pl->g.D ? pl->g.M : pl->g.M + 2;
        t.lo[ax] = 0;
        const int te = ax == 2 ? t.Tz : t.T;
        t.nt[ax] = (extent + te - 1) / te;
    }
}

static void bin_tiles(se_plan *pl, const double *pos, const double *q, int64_t N) {
    tile_setup(pl);
    TileGeom &t = pl->tile;
    int nbins = t.nt[0] * t.nt[1] * t.nt[2];
    binning_reserve(pl, pl->tbin, N, nbins, kUnit);
    prof_begin(pl, SE_K_SORT);
    SE_CUDA(cudaMemsetAsync(pl->tbin.counts.ptr, 0, sizeof(int) * (nbins + 1), pl->stream));
    SpreadArgs a = make_args(pl);
    if (N > 0 && nbins <= kTileHistSmem) {
        int64_t blocks = (N + 4095) / 4096;  // ~16 particles per thread
        if (blocks > 1184) blocks = 1184;
        tile_keys_hist_kernel<<<(unsigned)blocks, 256, sizeof(int) * nbins, pl->stream>>>(
            pos, N, a, nbins, pl->tbin.keys.as<unsigned>(), pl->tbin.counts.as<int>());
        SE_LAUNCH_CHECK();
        pl->launches += 1;
    } else if (N > 0) {
        tile_keys_kernel<<<(unsigned)((N + 255) / 256), 256, 0, pl->stream>>>(pos, N, a, pl->tbin.keys.as<unsigned>(),
                                                                               pl->tbin.counts.as<int>());
        SE_LAUNCH_CHECK();
        pl->launches += 1;
    }
    binning_sort(pl, pl->tbin, pos, q, N, nbins, kUnit);
    prof_end(pl, SE_K_SORT);
}

// compile-time window support for the common even P (others: runtime P)
template <class F>
static void dispatch_p(int P, F f) {
    switch (P) {
        case 4: f(std::integral_constant<int, 4>()); break;
        case 6: f(std::integral_constant<int, 6>()); break;
        case 8: f(std::integral_constant<int, 8>()); break;
        case 10: f(std::integral_constant<int, 10>()); break;
        case 12: f(std::integral_constant<int, 12>()); break;
        case 14: f(std::integral_constant<int, 14>()); break;
        case 16: f(std::integral_constant<int, 16>()); break;
        default: f(std::integral_constant<int, 0>()); break;
    }
}

template <class F>
static void dispatch_window(int window, F f) {
    if (window == SE_WINDOW_GAUSSIAN)
        f(std::integral_constant<int, SE_WINDOW_GAUSSIAN>());
    else if (window == SE_WINDOW_KB)
        f(std::integral_constant<int, SE_WINDOW_KB>());
    else
        f(std::integral_constant<int, SE_WINDOW_BM>());
}

static void shard_range(int64_t N, int rank, int world, int64_t &lo, int64_t &hi) {
    lo = N * rank / world;
    hi = N * (rank + 1) / world;
}

// SE_B200_SPREAD_WS=0 selects the single-role spreading kernel (A/B runs)
static bool spread_ws_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("SE_B200_SPREAD_WS");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

void spread_run(se_plan *pl, const double *pos, const double *q, int64_t N, double *grid, int rank, int world) {
    if (pl->p.P > pl->g.M) fail(SE_EINVAL, "window support P must not exceed M");
    const se_grid_t &g = pl->g;
    size_t gsize = (size_t)g.shape[0] * g.shape[1] * g.shape[2];
    tile_setup(pl);
    const bool det = pl->deterministic && pl->tile.T > 0;
    if (!det || N <= 0) SE_CUDA(cudaMemsetAsync(grid, 0, sizeof(double) * gsize, pl->stream));
    if (N <= 0) return;
    bin_tiles(pl, pos, q, N);
    SpreadArgs a = make_args(pl);
    shard_range(N, rank, world, a.rlo, a.rhi);
    const TileGeom &t = pl->tile;
    const double4 *rec = pl->tbin.rec.as<double4>();
    prof_begin(pl, SE_K_SPREAD);
    if (t.T > 0) {
        int64_t maxu = binning_max_units(pl->tbin, N, t.nt[0] * t.nt[1] * t.nt[2], kUnit);
        const int PC = t.nwarps == pl->p.P ? pl->p.P : 0;
        double *dbuf = nullptr;
        if (det) {
            pl->sdet.ensure(sizeof(double) * (size_t)maxu * t.Tp * t.Tp * t.pitch);
            dbuf = pl->sdet.as<double>();
        }
        if (PC == 8 && !det && spread_ws_enabled() && t.T == TileC<8>::T) {
            const size_t smem = t.smem + spread_ws_extra(8);
            dispatch_window(pl->p.window, [&](auto W) {
                auto kern = spread_ws_kernel<decltype(W)::value>;
                SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                kern<<<(unsigned)maxu, 32 * (kSwsC + kSwsP), smem, pl->stream>>>(rec, pl->tbin.units.as<int4>(),
                                                                                  pl->tbin.nunits.as<int>(), a, grid);
            });
        } else
        dispatch_window(pl->p.window, [&](auto W) {
            dispatch_p(PC, [&](auto PCv) {
                auto kern = spread_tile_kernel<decltype(W)::value, decltype(PCv)::value>;
                SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem));
                kern<<<(unsigned)maxu, 32 * t.nwarps, t.smem, pl->stream>>>(rec, pl->tbin.units.as<int4>(),
                                                                             pl->tbin.nunits.as<int>(), a, grid, dbuf);
            });
        });
        if (det) {
            SE_LAUNCH_CHECK();
            pl->launches += 1;
            spread_det_reduce_kernel<<<(unsigned)std::min<int64_t>((gsize + 255) / 256, 148 * 16), 256, 0,
                                       pl->stream>>>(dbuf, pl->tbin.units.as<int4>(), pl->tbin.ubstart.as<int>(), a,
                                                     (int64_t)gsize, grid);
        }
    } else {
        int64_t n = a.rhi - a.rlo;
        int wpb = 4;
        size_t sm = sizeof(double) * 3 * pl->p.P * wpb;
        dispatch_window(pl->p.window, [&](auto W) {
            auto kern = direct_kernel<decltype(W)::value, true>;
            SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            kern<<<(unsigned)((n + wpb - 1) / wpb), 32 * wpb, sm, pl->stream>>>(
                rec, pl->tbin.idx_sorted.as<int>(), a.rlo, a.rhi, a, grid, nullptr, nullptr, 0.0, 0);
        });
    }
    SE_LAUNCH_CHECK();
    prof_end(pl, SE_K_SPREAD);
    pl->launches += 1;
}

void gather_run(se_plan *pl, const double *grid, const double *pos, int64_t N, double *phi, int accumulate,
                int rank, int world, bool rebin) {
    if (N <= 0) return;
    // the fused pipelines reuse the spreading bins (same positions); a
    // stand-alone gather bins its own positions (charges are not read)
    if (rebin) bin_tiles(pl, pos, nullptr, N);
    SpreadArgs a = make_args(pl);
    int64_t lo, hi;
    shard_range(N, rank, world, lo, hi);
    a.rlo = lo;
    a.rhi = hi;
    if (!accumulate && world > 1) SE_CUDA(cudaMemsetAsync(phi, 0, sizeof(double) * N, pl->stream));
    const TileGeom &t = pl->tile;
    const double h3 = pl->g.h * pl->g.h * pl->g.h;
    const double4 *rec = pl->tbin.rec.as<double4>();
    prof_begin(pl, SE_K_GATHER);
    if (t.T > 0) {
        int64_t maxu = binning_max_units(pl->tbin, N, t.nt[0] * t.nt[1] * t.nt[2], kUnit);
        const int PC = t.nwarps == pl->p.P ? pl->p.P : 0;
        dispatch_window(pl->p.window, [&](auto W) {
            dispatch_p(PC, [&](auto PCv) {
                auto kern = gather_tile_kernel<decltype(W)::value, decltype(PCv)::value>;
                SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem));
                kern<<<(unsigned)maxu, 32 * t.nwarps, t.smem, pl->stream>>>(
                    rec, pl->tbin.idx_sorted.as<int>(), pl->tbin.units.as<int4>(), pl->tbin.nunits.as<int>(), a, grid,
                    phi, h3, accumulate);
            });
        });
    } else {
        int64_t n = a.rhi - a.rlo;
        int wpb = 4;
        size_t sm = sizeof(double) * 3 * pl->p.P * wpb;
        dispatch_window(pl->p.window, [&](auto W) {
            auto kern = direct_kernel<decltype(W)::value, false>;
            SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            kern<<<(unsigned)((n + wpb - 1) / wpb), 32 * wpb, sm, pl->stream>>>(
                rec, pl->tbin.idx_sorted.as<int>(), a.rlo, a.rhi, a, nullptr, grid, phi, h3, accumulate);
        });
    }
    SE_LAUNCH_CHECK();
    prof_end(pl, SE_K_GATHER);
    pl->launches += 1;
}

// ------------------------------------------- gradient gather (E = -grad phi_F)
// Derivative of the window (windows.py:74-84, 106-112): Gaussian
// w' = 2 gcoef x w; Kaiser-Bessel w' = -beta I1(beta s) r / (w s I0(beta)),
// s = sqrt(1 - r^2), r = x / w (I1(beta s) / s -> beta / 2 at the support
// edge: finite).  The ES window's derivative is singular at the edge and
// is not used here (the D = 3 field differentiates spectrally instead).
template <int WIN>
__device__ __forceinline__ double window_deriv(double x, const SpreadArgs &a) {
    if (!(fabs(x) <= a.w)) return 0.0;
    if (WIN == SE_WINDOW_GAUSSIAN) return 2.0 * a.gcoef * x * (a.peak * exp_nonpos(a.gcoef * (x * x)));
    const double r = x * a.invw;
    double t = fma(-r, r, 1.0);
    t = t < 0.0 ? 0.0 : t;
    const double sq = sqrt(t), z = a.shapep * sq;
    const double i1_over_s = sq > 1e-8 ? cyl_bessel_i1(z) / sq : 0.5 * a.shapep;
    return -a.shapep * i1_over_s * r * a.invw / a.i0b;
}

// One warp per particle (sorted by tile, so that neighbouring warps share
// grid lines in L2): E_a = h^3 sum_g H[g] w'(delta_a) prod_{b != a} w(delta_b)
// with delta = g h - (x + offset) -- the gradient of sekspace.gather's
// h^3 sum H w w w (sekspace.py:159-178) with respect to the particle position.
template <int WIN>
__global__ void __launch_bounds__(128) grad_gather_kernel(const double4 *__restrict__ rec, const int *__restrict__ sidx,
                                                         int64_t N, SpreadArgs a, const double *__restrict__ grid,
                                                         double *__restrict__ E, double h3, int accumulate) {
    extern __shared__ double gsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int P = a.P;
    double *w = gsm + warp * 6 * P;                      // w[axis][t], then dw[axis][t]
    int *gi = reinterpret_cast<int *>(gsm + nw * 6 * P) + warp * 3 * P;  // grid index per axis and t (-1: off)
    for (int64_t p = blockIdx.x * (int64_t)nw + warp; p < N; p += (int64_t)gridDim.x * nw) {
        const double4 r = rec[p];
        for (int task = lane; task < 3 * P; task += 32) {
            const int ax = task / P, t = task - ax * P;
            const double x = ax == 0 ? r.x : (ax == 1 ? r.y : r.z);
            const double u = __dadd_rn(x, a.off[ax]);
            const long long f = stencil_first(u, a) + t;
            const double d = __dsub_rn(__dmul_rn((double)f, a.h), u);  // sekspace.py:116
            w[ax * P + t] = window_eval<WIN>(d, a);
            w[(3 + ax) * P + t] = window_deriv<WIN>(d, a);
            long long g = f;
            if (ax < a.D) {
                g %= a.M;
                if (g < 0) g += a.M;
            } else if (g < 0 || g >= a.Mt) {
                g = -1;
            }
            gi[ax * P + t] = (int)g;
        }
        __syncwarp();
        double ex = 0.0, ey = 0.0, ez = 0.0;
        for (int pi = lane; pi < P * P; pi += 32) {
            const int ty = pi / P, tz = pi - ty * P;
            const int gy = gi[P + ty], gz = gi[2 * P + tz];
            if (gy < 0 || gz < 0) continue;
            double s = 0.0, sd = 0.0;
            for (int t = 0; t < P; ++t) {
                const int gx = gi[t];
                if (gx < 0) continue;
                const double c = grid[((int64_t)gx * a.shape[1] + gy) * a.shape[2] + gz];
                s = fma(w[t], c, s);
                sd = fma(w[3 * P + t], c, sd);
            }
            const double wy = w[P + ty], wz = w[2 * P + tz];
            ex = fma(wy * wz, sd, ex);
            ey = fma(w[4 * P + ty] * wz, s, ey);
            ez = fma(wy * w[5 * P + tz], s, ez);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ex += __shfl_xor_sync(0xffffffffu, ex, o);
            ey += __shfl_xor_sync(0xffffffffu, ey, o);
            ez += __shfl_xor_sync(0xffffffffu, ez, o);
        }
        if (lane == 0) {
            double *o = E + 3 * (int64_t)sidx[p];
            o[0] = accumulate ? o[0] + h3 * ex : h3 * ex;
            o[1] = accumulate ? o[1] + h3 * ey : h3 * ey;
            o[2] = accumulate ? o[2] + h3 * ez : h3 * ez;
        }
        __syncwarp();
    }
}

void grad_gather_run(se_plan *pl, const double *grid, const double *pos, int64_t N, double *E, int accumulate) {
    if (N <= 0) return;
    if (pl->p.window == SE_WINDOW_BM)
        fail(SE_EINVAL, "the window-gradient field needs the Gaussian or Kaiser-Bessel window (the ES window's "
                        "derivative is singular at its support edge)");
    bin_tiles(pl, pos, nullptr, N);
    SpreadArgs a = make_args(pl);
    const double h3 = pl->g.h * pl->g.h * pl->g.h;
    const int wpb = 4;
    const size_t sm = (sizeof(double) * 6 + sizeof(int) * 3) * (size_t)pl->p.P * wpb;
    int64_t blocks = (N + wpb - 1) / wpb;
    if (blocks > 148 * 32) blocks = 148 * 32;
    prof_begin(pl, SE_K_GATHER);
    dispatch_window(pl->p.window, [&](auto W) {
        auto kern = grad_gather_kernel<decltype(W)::value>;
        SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        kern<<<(unsigned)blocks, 32 * wpb, sm, pl->stream>>>(pl->tbin.rec.as<double4>(), pl->tbin.idx_sorted.as<int>(),
                                                             N, a, grid, E, h3, accumulate);
    });
    SE_LAUNCH_CHECK();
    prof_end(pl, SE_K_GATHER);
    pl->launches += 1;
}

}  // namespace se
