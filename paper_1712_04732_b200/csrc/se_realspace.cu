// Real-space Ewald sum and self term: realspace.real_space_sum /
// realspace.self_term (realspace.py:91-185).
//
// phi_R(x_t) = sum_{s, image p, |x_t - x_s + p| < rc, r >= 1e-14} q_s erfc(xi r)/r
//
// Column path (rc <= L/2 on periodic axes, or any rc for free axes):
//  * particles binned into columns (cx, cy) of edge >= rc/3 in x and y and
//    sorted by z inside each column (a 32-bit key: column, quantized z), as
//    (x, y, z, q) double4 records -- the reference bins into rc-edge cells
//    (build_cell_list, realspace.py:43-59);
//  * one warp per unit = 16 consecutive targets of a column (a thin z-slab);
//  * for each neighbour column within +-3 (half shell with Newton's third
//    law), the z-window that can hold partners, |dz| <= sqrt(rc^2 - gap^2)
//    around the slab, is found by a binary search in the column (one lane per
//    column, all columns of the half shell at once), and only that run is
//    streamed (~2.1x the in-cutoff pairs instead of
//    ~3.7x for 5x5x5 rc/2 cells); periodic z adds the window's wrapped parts
//    as shifted images;
//  * sources are staged 32 at a time in the warp's shared workspace with the
//    image shift folded in; an fp32 prefilter + warp compaction + exact fp64
//    evaluation follows (see pair_batch);
//  * periodic x/y with fewer than 7 columns visit every column once and use
//    the minimum image per pair (the reference's (cell, shift) de-duplication
//    for small n, realspace.py:98-109, gives the same pair set).
// Image path (D >= 1 and rc > L/2): all pairs x explicit images
// (realspace.py:138-165), one thread per target.
#include <algorithm>
#include <vector>

#include "se_common.h"
#include "se_erfc_coeffs.h"

namespace se {

struct RealArgs {
    int n;           // cells per axis
    double edge, L, xi, rc, rc2;
    int mode[3];     // 0 free, 1 periodic +-2 wrap, 2 periodic all cells + min image
    int64_t rlo, rhi;
    int add_self;
    double sqrtpi;
    float rc2f;       // fp32 prefilter bound (rc^2 plus the fp32 coordinate rounding margin)
    float Lf, invLf;  // box length for the fp32 minimum image
    int kb;           // bits of the z key (particles of a column sorted by z)
    double qinv;      // z quantum^-1 = 2^kb / L: Q(z) = floor(z qinv), monotone along a column
    int zper;         // z periodic (D = 3)
    int reach;        // neighbour columns within +-reach (column edge >= rc / reach)
    int dense_min;    // prefilter hits per full batch (of kT x 32) from which the batch is
                      // evaluated densely (all pairs, no compaction); > kT * 32: never
    int64_t n_own;    // domain mode: caller-order particles [0, n_own) get the self term; -1: off
    // Polynomial pair term (kernels with DEG > 0, see pair_poly):
    //   erfc(xi r)/r = 1/r - Q(r^2),  Q(u) = sum_i pc[i] t^i,  t = u pscale - 1
    double rc2x;               // rc^2: the exact cutoff test r^2 < rc^2
    double pscale;             // 2 / rc^2: u in [0, rc^2] -> t in [-1, 1]
    double pc[33];             // monomial coefficients in t (degree <= 32)
    int pdeg;                  // host: degree fitted (0: use erfc_fast)
};

constexpr double kTwoOverSqrtPi = 1.1283791670955126;  // field mode: c = 2 xi / sqrt(pi)

// columns of edge >= rc/reach: neighbours within +-reach columns; reach 3
// (fewer candidates) unless columns would be short (small N: every visited
// column costs at least one batch, so fewer, longer columns win)
constexpr int kReachMax = 3;
constexpr double kShortColumn = 256.0;  // mean particles per column below which reach = 2

__device__ __forceinline__ int zq(double z, double qinv) { return (int)floor(z * qinv); }

// fp32 prefilter bound: coordinates in [-L, 2L) carry <= 2^-23 L absolute
// rounding each, so r^2 in fp32 is within ~1.5e-6 rc L (+ fp32 products) of
// the exact value for candidates near the cutoff; 4x that keeps every pair
// with r < rc.
static inline void set_prefilter(RealArgs &a) {
    a.rc2f = (float)(a.rc * a.rc + 6e-6 * a.rc * a.L + 2e-6 * a.rc * a.rc);
    a.Lf = (float)a.L;
    a.invLf = (float)(1.0 / a.L);
}

__device__ __forceinline__ unsigned column_key(const double *__restrict__ pos, int64_t i, const RealArgs &a,
                                               unsigned &colid) {
    int c[2];
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
        // clamped on both sides: the C ABI rejects coordinates outside
        // [0, L), this only keeps an unchecked caller's keys in range
        int ci = (int)floor(sane_coord(pos[3 * i + ax], a.L, i, ax) / a.edge);
        ci = ci < 0 ? 0 : ci;
        c[ax] = ci < a.n - 1 ? ci : a.n - 1;
    }
    colid = (unsigned)(c[0] * a.n + c[1]);
    // within a column, order by the quantized z: Q(z) = floor(z qinv) is then
    // non-decreasing along every column (z in [0, L))
    int sub = zq(sane_coord(pos[3 * i + 2], a.L, i, 2), a.qinv);
    sub = sub < 0 ? 0 : (sub >= (1 << a.kb) ? (1 << a.kb) - 1 : sub);
    return (colid << a.kb) | (unsigned)sub;
}

__global__ void cell_keys_kernel(const double *__restrict__ pos, int64_t N, RealArgs a, unsigned *__restrict__ keys,
                                 int *__restrict__ counts) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    unsigned colid;
    keys[i] = column_key(pos, i, a, colid);
    atomicAdd(&counts[colid], 1);
}

// Few columns (<= kHistSmem): per-block shared-memory histogram, flushed
// once per non-empty column (~1000 particles per column contend on one
// global counter otherwise).
constexpr int kHistSmem = 8192;
__global__ void cell_keys_hist_kernel(const double *__restrict__ pos, int64_t N, RealArgs a, int nbins,
                                      unsigned *__restrict__ keys, int *__restrict__ counts) {
    extern __shared__ int hist[];
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned colid;
        keys[i] = column_key(pos, i, a, colid);
        atomicAdd(&hist[colid], 1);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nbins; b += blockDim.x)
        if (hist[b]) atomicAdd(&counts[b], hist[b]);
}

// Scalar constants of erfc_fast as one constant-bank block (read two per
// LDCU.128 instead of materialised as 64-bit immediates per use).
__constant__ double se_erfc_k[6] = {
    SE_ERFC_A + SE_ERFC_B,                // s = ((A+B) x + K (B-A)) / (x + K)
    SE_ERFC_K * (SE_ERFC_B - SE_ERFC_A),  //   (K = 4: an immediate)
    -SE_LOG2E,                            // n = rint(-x^2 log2 e) by the 1.5 2^52 shifter
    -SE_LN2_HI,                           // r = -x^2 - n ln2 (one rounded ln2, see exp_neg)
    6755399441055744.0,                   // 1.5 2^52
    0.375};                               // rsqrt_nr: a 64-bit constant operand, not
                                          //   two IMAD.MOVs per use

// 1/d and 1/sqrt(d): the MUFU approximations (~2^-22 relative) and one
// third-order correction each (error O(e^3): ~1 ulp), branch-free; d is a
// positive normal number here.
__device__ __forceinline__ double rcp_nr(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double e = fma(-d, y, 1.0);  // 1/d = y / (1 - e) = y (1 + e + e^2 + ...)
    return fma(y, fma(e, e, e), y);
}
__device__ __forceinline__ double rsqrt_nr(double d) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double e = fma(-d * y, y, 1.0);  // d^-1/2 = y (1 - e)^-1/2 = y (1 + e/2 + 3e^2/8 + ...)
    return fma(y, e * fma(e, se_erfc_k[5], 0.5), y);
}

// exp(-u) for 0 <= u <= ~40 as e 2^n: returns the reduced factor e in
// [2^-1/2, 2^1/2] and n (<= 0).  n = rint(-u log2 e) by the 1.5 2^52
// shifter (one DFMA and one DADD; n is the low word -- no FRND / F2I), and
// r = -u - n ln2 with ONE rounded ln2 (one DFMA instead of the two of a
// Cody-Waite split): the ln2 rounding moves r by |n| 2^-53 ln2, a relative
// error of exp(-u) of at most 1.1e-16 u, i.e. an absolute error of
// erfc(x) = exp(-u) erfcx(x) below 1.1e-16 u erfc(sqrt u) <= 1.7e-17 --
// under the erfcx fit's own 7.6e-17.
__device__ __forceinline__ double exp_neg(double u, int &n) {
    const double t = fma(u, se_erfc_k[2], se_erfc_k[4]);
    n = __double2loint(t);
    const double nf = t - se_erfc_k[4];
    const double r = fma(nf, se_erfc_k[3], -u);
    double e = se_exp_c[SE_EXP_NX];
#pragma unroll
    for (int i = SE_EXP_NX - 1; i >= 2; --i) e = fma(e, r, se_exp_c[i]);
    return fma(fma(e, r, SE_EXP_C1), r, SE_EXP_C0);  // literals (1.0): no constant-bank operands
}

// e 2^n by an exponent add (n in [-60, 0] and e ~ 1: e 2^n stays normal)
__device__ __forceinline__ double scale2(double e, int n) {
    return __hiloint2double(__double2hiint(e) + n * (1 << 20), __double2loint(e));
}

// erfc(x), x >= 0, as exp(-x^2) erfcx(x): erfcx by a degree-14 polynomial in
// s = A t + B, t = (x - K)/(x + K), and exp by exp_neg; coefficients are
// __constant__ operands (tools/gen_erfc_coeffs.py: fitted for absolute
// accuracy, max error 7.6e-17 absolute / 7.6e-10 relative on [0, 6] -- the
// pair term's 1/r rounding is ~1e-16 relative).  The x^2 rounding residual
// is not carried: it moves exp(-x^2) by <= x^2 2^-53 relative, i.e. <= 4e-17
// absolute, below the 1/r rounding of the pair term.  Beyond SE_ERFC_XMAX
// the library erfc is used.
//
// erfc(x) * w.  WIDE: x may exceed SE_ERFC_XMAX (xi rc > 6, i.e. eps < 2e-16).
// Otherwise the caller guarantees x <= SE_ERFC_XMAX (1 + 1e-4) for every
// evaluated pair (beyond the cutoff the result is multiplied by w = 0), and
// the code is branch-free so that two evaluations form one basic block the
// scheduler can interleave.
template <bool WIDE>
__device__ __forceinline__ double erfc_fast(double x, double w) {
    if (WIDE) {
        if (x > SE_ERFC_XMAX) return erfc(x) * w;
    }
    const double s = fma(x, se_erfc_k[0], se_erfc_k[1]) * rcp_nr(x + SE_ERFC_K);
    // Horner (Estrin's shorter chains measured slower: the kernel is
    // issue bound)
    double p = se_erfcx_c[SE_ERFC_NE];
#pragma unroll
    for (int i = SE_ERFC_NE - 1; i >= 0; --i) p = fma(p, s, se_erfcx_c[i]);
    int n;
    const double e = exp_neg(x * x, n);
    return p * (scale2(e, n) * w);
}

// Field mode: the two factors separately, erfcx(x) (as p) and exp(-x^2) (as
// e): E_R needs erfc(x)/r + (2 xi / sqrt(pi)) exp(-x^2) = e (p / r + c).
template <bool WIDE>
__device__ __forceinline__ void erfc_parts(double x, double &p, double &e) {
    if (WIDE) {
        if (x > SE_ERFC_XMAX) {
            p = erfcx(x);
            e = exp(-x * x);
            return;
        }
    }
    const double s = fma(x, se_erfc_k[0], se_erfc_k[1]) * rcp_nr(x + SE_ERFC_K);
    p = se_erfcx_c[SE_ERFC_NE];
#pragma unroll
    for (int i = SE_ERFC_NE - 1; i >= 0; --i) p = fma(p, s, se_erfcx_c[i]);
    int n;
    e = scale2(exp_neg(x * x, n), n);
}

// Pair term without exp / erfc: erfc(xi r)/r = 1/r - xi erf(xi r)/(xi r), and
// erf(x)/x is an entire function of x^2 = xi^2 u, so on u in [0, rc^2] it is a
// single polynomial in t = u (2/rc^2) - 1 (degree DEG, fitted per plan by
// fit_pair_poly: Chebyshev interpolant of xi erf(xi sqrt u)/(xi sqrt u) in
// long double, truncation error below 2e-16 / rc -- the rounding of 1/r at
// the cutoff; its monomial coefficients are < 1 in magnitude, so Horner in
// fp64 is well conditioned).  Compared with erfc_fast (a rational transform,
// a reciprocal, erfcx and exp polynomials, an exponent scale) this is one
// DFMA for t, DEG DFMAs and one DADD: no MUFU.RCP, no integer work.  The
// result is exact to the rounding of 1/r plus ~2 ulp of Q in ABSOLUTE terms
// (the subtraction cancels towards the cutoff, where the term is ~eps/rc).
// Valid for u in [0, rc^2]; outside, the caller discards the value.
template <int DEG>
__device__ __forceinline__ double pair_poly(double u, const RealArgs &a) {
    const double y = rsqrt_nr(u);
    const double t = fma(u, a.pscale, -1.0);
    double p = a.pc[DEG];
#pragma unroll
    for (int i = DEG - 1; i >= 0; --i) p = fma(p, t, a.pc[i]);
    return y - p;
}

__device__ __forceinline__ double min_image(double d, double L) { return d - L * rint(d / L); }
__device__ __forceinline__ float min_image_f(float d, float L, float invL) { return d - L * rintf(d * invL); }

constexpr int kWarps = 1;  // warps (units) per block: one, so that the WarpBuf base is
                           // block-uniform (shared addresses fold into [R + UR + imm])
#ifndef SE_RS_MINBLOCKS
#define SE_RS_MINBLOCKS 27
#endif
constexpr int kMinBlocks = SE_RS_MINBLOCKS;  // 27 x (7 KB + 1 KB reserved) of shared memory per SM
constexpr int kT = 16;     // targets per warp unit: lane l tests target l % 16 against half of a 32-source batch
constexpr int kDenseMin = 410;  // ~0.8 kT x 32: dense evaluation of a batch from this many prefilter hits

// Shared-memory workspace of one warp unit (7 KB; 15 KB in field mode, FLD:
// three accumulator components).
template <bool FLD>
struct __align__(16) WarpBufT {
    double2 txy[kT], tzq[kT];    // the unit's targets: (x, y), (z, q) -- one LDS.128 each
    double2 sxy[32], szq[32];    // current source batch, likewise (16-B stride: a warp's
                                 // random reads cost the minimum 4 wavefronts per LDS.128)
    float4 sf[32];               // the same in fp32 for the prefilter
    float4 tf[kT];               // unit targets relative to the unit origin, fp32 (w: 1 if inactive)
    double acc[FLD ? 3 : 1][kT][32];  // per-lane private accumulators acc[c][t][lane]: lane-owned banks
    unsigned short ent[kT * 32];  // compacted hits of a batch: (target slot << 5) | source
};
// field mode: 13 CTAs x (15 KB + 1 KB reserved) per SM
constexpr int kMinBlocksField = 13;

// Shared-memory slot of unit target t: targets t and t + 8 (one prefilter
// lane's pair) land in different bank quads of txy / tzq (slot t ^ 4 for
// t >= 8), so a quarter warp's LDS.128 of its hits' targets is conflict
// free (with slot = t it was 2-way: 7.9 wavefronts per load instead of 4).
// Entries and acc rows are indexed by slot.
__device__ __forceinline__ int tslot(int t) { return t ^ ((t >> 3) << 2); }

// Fire-and-forget L1 prefetch of a record the warp stages later (the staging
// load otherwise waits a full L2 round trip per batch).
__device__ __forceinline__ void prefetch_l1(const double4 *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// Exact fp64 evaluation of one compacted hit (target tt, source k of the
// batch): d = x_t - (x_s + shift) (realspace.py:113-117), the coincidence
// check (r < 1e-14, realspace.py:118-122), r < rc, and f = erfc(xi r)/r with
// 1/r = rsqrt(r^2).  Branch-free; the caller applies the result.
struct Hit {
    double f;   // erfc(xi r)/r, 0 outside the cutoff
    double qt;  // target charge (source-side update with NEWTON)
    double qs;  // source charge (target-side update)
    double dx, dy, dz;  // x_t - x_s (field mode)
    double u;           // r^2 as evaluated (field mode, polynomial pair term)
    int tt, k;
    bool ok;
};

// Geometry of one hit up to the erfc argument: h.f = w (1/r, or 0 outside
// the cutoff or for an invalid slot), returns x = xi r.
template <bool MI, bool NEWTON, bool FLD, class WB>
__device__ __forceinline__ double hit_geometry(unsigned en, bool valid, const RealArgs &a, const WB &wb, int jb,
                                               int tbase, int &singular, Hit &h) {
    h.tt = (int)(en >> 5);
    h.k = (int)(en & 31u);
    const double2 t01 = wb.txy[h.tt], t23 = wb.tzq[h.tt];
    const double2 s01 = wb.sxy[h.k], s23 = wb.szq[h.k];
    double dx = t01.x - s01.x, dy = t01.y - s01.y, dz = t23.x - s23.x;
    if (MI) {
        if (a.mode[0] == 2) dx = min_image(dx, a.L);
        if (a.mode[1] == 2) dy = min_image(dy, a.L);
        if (a.mode[2] == 2) dz = min_image(dz, a.L);
    }
    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
    // r < 1e-14: the self pair (never compacted with NEWTON) or a coincidence
    const bool zero = r2 < 1e-28;
    double r2s;
    if (NEWTON) {
        // any zero distance is a coincidence: the call raises and its
        // result (here NaN for r = 0) is discarded -- no select needed
        singular |= zero ? 1 : 0;
        r2s = r2;
    } else {
        singular |= (zero && jb + h.k != tbase + tslot(h.tt)) ? 1 : 0;
        r2s = zero ? a.rc2 : r2;  // the self pair: evaluated at r = rc and dropped
    }
    const double rinv = rsqrt_nr(r2s);
    const double rr = r2s * rinv;
    h.ok = valid && rr < a.rc && (NEWTON || !zero);
    h.f = h.ok ? rinv : 0.0;  // a select, not a branch: the erfc runs unconditionally
    h.qt = t23.y;
    h.qs = s23.y;
    if (FLD) {
        h.dx = dx;
        h.dy = dy;
        h.dz = dz;
        h.u = r2s;
    }
    return a.xi * rr;
}

// Potential mode: h.f = erfc(x) w.  Field mode (FLD): h.f = g with
// E_t += q_s g (x_t - x_s), g = (erfc(x)/r + c exp(-x^2)) / r^2 =
// e w^2 (p w + c), c = 2 xi / sqrt(pi) (w = 1/r, 0 outside the cutoff).
template <bool WIDE, bool FLD>
__device__ __forceinline__ void hit_value(double x, const RealArgs &a, Hit &h) {
    if (FLD) {
        double p, e;
        erfc_parts<WIDE>(x, p, e);
        const double w = h.f;
        h.f = e * (w * w) * fma(p, w, a.xi * kTwoOverSqrtPi);
    } else {
        h.f = erfc_fast<WIDE>(x, h.f);
    }
}

// Field mode with the polynomial pair term: g = (erfc(x)/r + c exp(-x^2))/r^2
// = w^2 (w - R(r^2)), R(u) = Q(u) - c exp(-xi^2 u) -- one entire function,
// fitted like Q (pair_poly_fit, kind 1); w = 1/r, or 0 outside the cutoff.
template <int DEG>
__device__ __forceinline__ void hit_value_field_poly(const RealArgs &a, Hit &h) {
    const double t = fma(h.u, a.pscale, -1.0);
    double p = a.pc[DEG];
#pragma unroll
    for (int i = DEG - 1; i >= 0; --i) p = fma(p, t, a.pc[i]);
    const double w = h.f;
    h.f = (w * w) * (w - p);
}

template <bool MI, bool NEWTON, bool WIDE, bool FLD, class WB>
__device__ __forceinline__ Hit eval_hit(unsigned en, const RealArgs &a, const WB &wb, int jb, int tbase,
                                        int &singular) {
    Hit h;
    const double x = hit_geometry<MI, NEWTON, FLD>(en, true, a, wb, jb, tbase, singular, h);
    hit_value<WIDE, FLD>(x, a, h);
    return h;
}

// Polynomial path (DEG > 0: NEWTON, no minimum image, potential): one
// compacted hit (slot tt, source k) -> h.f = erfc(xi r)/r, 0 outside the
// cutoff or for an invalid (duplicate) slot.  Any zero distance among the
// hits is a coincidence (the self pair is never compacted with NEWTON).
// Without NEWTON (the deterministic mode's full shell) the prefilter also
// passes the self pair (source jb + k == target tbase + t): dropped, not flagged.
template <int DEG, bool NEWTON = true, class WB>
__device__ __forceinline__ void hit_poly(unsigned en, bool valid, const RealArgs &a, const WB &wb, int &singular,
                                         Hit &h, int jb = 0, int tbase = 0) {
    h.tt = (int)(en >> 5);
    h.k = (int)(en & 31u);
    const double2 t01 = wb.txy[h.tt], t23 = wb.tzq[h.tt];
    const double2 s01 = wb.sxy[h.k], s23 = wb.szq[h.k];
    const double dx = t01.x - s01.x, dy = t01.y - s01.y, dz = t23.x - s23.x;
    const double u = fma(dz, dz, fma(dy, dy, dx * dx));
    // u >= 0: the order of its bit pattern is the order of its value, so both
    // tests run on the integer pipe (a DSETP occupies the fp64 pipe)
    const long long ub = __double_as_longlong(u);
    const bool zero = ub < 0x3A1FB0F6BE506019LL;  // u < 1e-28
    if (NEWTON) {
        singular |= zero ? 1 : 0;
        h.ok = valid && ub < __double_as_longlong(a.rc2x);
    } else {
        singular |= (valid && zero && jb + h.k != tbase + tslot(h.tt)) ? 1 : 0;
        h.ok = valid && !zero && ub < __double_as_longlong(a.rc2x);
    }
    const double f = pair_poly<DEG>(u, a);
    h.f = h.ok ? f : 0.0;
    h.qt = t23.y;
    h.qs = s23.y;
}

// Target side into the lane's private slot; with NEWTON the source side
// q_t f goes to the source's global accumulator (REDG).
// Field mode: three components on both sides (the source side with the
// opposite sign), acc_batch in (3 j + c) layout.
template <bool NEWTON, bool FLD>
__device__ __forceinline__ void apply_hit(const Hit &h, WarpBufT<FLD> &wb, int lane, double *__restrict__ acc_batch) {
    if (FLD) {
        const double gs = h.qs * h.f;
        double *s0 = &wb.acc[0][h.tt][lane], *s1 = &wb.acc[FLD ? 1 : 0][h.tt][lane],
               *s2 = &wb.acc[FLD ? 2 : 0][h.tt][lane];
        *s0 = fma(gs, h.dx, *s0);
        *s1 = fma(gs, h.dy, *s1);
        *s2 = fma(gs, h.dz, *s2);
        if (NEWTON && h.ok) {
            const double gt = -h.qt * h.f;
            atomicAdd(acc_batch + 3 * h.k, gt * h.dx);
            atomicAdd(acc_batch + 3 * h.k + 1, gt * h.dy);
            atomicAdd(acc_batch + 3 * h.k + 2, gt * h.dz);
        }
        return;
    }
    double *slot = &wb.acc[0][h.tt][lane];
    *slot = fma(h.qs, h.f, *slot);
#ifdef SE_AB_NO_REDG  // timing experiment only (wrong results): no source-side reductions
    if (NEWTON && h.ok && h.f == 123.0) atomicAdd(acc_batch + h.k, h.qt * h.f);
#else
    if (NEWTON && h.ok) atomicAdd(acc_batch + h.k, h.qt * h.f);
#endif
}

// Packed fp32x2 arithmetic (FFMA2 / FADD2, sm_100): two prefilter tests per
// instruction, the scalar source operand broadcast to both lanes of the pair.
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, float b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(f2pack(b, b)), "l"(c));
    return r;
}
__device__ __forceinline__ unsigned long long f2add(unsigned long long a, float b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(f2pack(b, b)));
    return r;
}

// Prefilter operands of one lane: targets pa = lane % 8 and pa + 8 of the
// unit (lo / hi halves of the packed pairs), sources 8 (lane / 8) .. + 7 of
// each batch.  Outside minimum-image mode: (-2 t'x, -2 t'y, -2 t'z,
// |t'|^2 - bound) with t' relative to org = (column corner, lowest target z); in it the
// absolute fp32 positions.  An absent target never passes.
struct PreTargets {
    unsigned long long x, y, z, w;
    int ta, tb;       // unit-relative target slots (pa, pa + 8)
    unsigned amask;   // bit t: unit target t is active (bits 16..31 repeat 0..15)
};

// Dense evaluation of a batch whose prefilter hit nearly every (target,
// source) slot (most batches in the middle of a column window): no
// compaction.  Lane l keeps source l of the batch in registers (staged by
// itself) and, in step s = 0..kT-1, pairs it with unit target (l + s) mod kT
// -- every (target, source) slot exactly once, the 32 lanes of a step on 32
// different sources and kT targets (two lanes per target, different
// acc columns).  The target side goes to the lane-owned slot acc[t][l]; the
// source side accumulates in a register and leaves with ONE REDG per source
// and batch (instead of one per pair).  Pairs outside the cutoff, excluded
// own-column pairs (j <= t), inactive targets and lanes past the run's end
// are evaluated at r = rc and multiplied by 0.  Newton (half-shell) path only.
template <bool WIDE, class WB>
__device__ __forceinline__ void dense_batch(WB &wb, int lane, int j, int m, double xs, double ys, double zs, double qs,
                                            const RealArgs &a, unsigned amask, int tbase, int hs, const double3 org,
                                            double *__restrict__ acc_s, int &singular) {
    const bool sval = lane < m;
    if (!sval) {  // past the run's end: a harmless nearby point (never counted)
        xs = org.x;
        ys = org.y;
        zs = org.z;
    }
    // valid (target, this source) pairs as a 16-bit mask over the target
    // SLOTS (tslot order), built once per batch: active targets, and in the
    // own column only targets t < j (the pair j <= t is visited from j's side)
    unsigned vt = amask & 0xffffu;
    if (hs >= 0) {
        const int c = min(max(j - tbase, 0), kT);
        vt &= (1u << c) - 1u;
    }
    if (!sval) vt = 0u;
    const unsigned vs = (vt & 0x00ffu) | ((vt & 0x0f00u) << 4) | ((vt & 0xf000u) >> 4);
    double accs = 0.0;
#pragma unroll 2
    for (int st = 0; st < kT; ++st) {
        const int sl = (lane + st) & (kT - 1);  // a slot; lanes l and l + 16 share it
        const double2 t01 = wb.txy[sl], t23 = wb.tzq[sl];
        const bool v = (vs >> sl) & 1u;
        const double dx = t01.x - xs, dy = t01.y - ys, dz = t23.x - zs;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const bool zero = r2 < 1e-28;
        singular |= (v && zero) ? 1 : 0;
        // a valid pair is a real pair of the column window (r <~ 2 rc: erfc_fast's
        // argument stays bounded; pairs beyond rc get w = 0); every other slot
        // (inactive target slots hold zeros, the self pair r = 0) is evaluated
        // at r = rc and dropped
        const bool use = v && !zero;
        const double r2s = use ? r2 : a.rc2;
        const double rinv = rsqrt_nr(r2s);
        const double rr = r2s * rinv;
        const double w = (use && rr < a.rc) ? rinv : 0.0;
        const double f = erfc_fast<WIDE>(a.xi * rr, w);
        double *slot = &wb.acc[0][sl][lane];
        *slot = fma(qs, f, *slot);
        accs = fma(t23.y, f, accs);
    }
    if (sval) atomicAdd(acc_s + lane, accs);
    __syncwarp();
}

// Dense batch, polynomial pair term (DEG > 0): lane l keeps source l in
// registers; step t pairs it with unit target t, the same for all lanes --
// the target is a broadcast shared-memory read (2 LDS.128 of one address)
// and its accumulator row acc[tslot(t)][lane] a lane-private slot.  Two
// targets per step, their polynomials as two interleaved Horner chains
// (one chain per warp is latency bound); a rolled loop keeps the code in
// the instruction cache.  Inactive target slots and sources past the run's
// end sit far away (r > rc), so outside the own column (OWN = false) the
// only test per slot is r^2 < rc^2 -- on the integer bits of r^2 (ALU, not
// the fp64 pipe), as is the coincidence test 1/r > 1e14 (r < 1e-14).  In
// the own column (OWN) only targets t < j count (the pair j <= t is visited
// from j's side).  The source side leaves with one REDG per source and batch.
__device__ __forceinline__ bool below_bits(double u, long long lim) { return __double_as_longlong(u) < lim; }

#ifndef SE_DENSE_NT
#define SE_DENSE_NT 2  // targets (interleaved Horner chains) per step
#endif
#ifndef SE_DENSE_UNROLL
#define SE_DENSE_UNROLL 1  // measured: 1 beats 2 by 2-4% (cfg2, cfg5, cfg4)
#endif
constexpr int kDenseUnroll = SE_DENSE_UNROLL;
// Without NEWTON (the full shell of the deterministic mode: every target sums
// all its partners, no source side) the own column (OWN) drops only the self
// pair t == j, and nothing leaves through atomics.
template <int DEG, bool OWN, bool NEWTON = true, class WB>
__device__ __forceinline__ void dense_batch_poly(WB &wb, int lane, int j, int m, double xs, double ys, double zs,
                                                 double qs, const RealArgs &a, unsigned amask, int tbase,
                                                 double *__restrict__ acc_s, int &singular) {
    constexpr int NT = SE_DENSE_NT;
    unsigned vt = 0xffffu;
    if (OWN) {
        if (NEWTON) {
            const int c = min(max(j - tbase, 0), kT);
            vt = amask & ((1u << c) - 1u);
        } else {
            const int c = j - tbase;
            vt = amask & ~((c >= 0 && c < kT) ? (1u << c) : 0u);
        }
    }
    const long long lim = __double_as_longlong(a.rc2x);  // r^2 >= 0: bit order = value order
    double accs = 0.0;
    bool sing = false;
#pragma unroll kDenseUnroll
    for (int t = 0; t < kT; t += NT) {
        int sl[NT];
        double2 p01[NT], p23[NT];
        double u[NT], y[NT], tv[NT], p[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            sl[k] = tslot(t + k);
            p01[k] = wb.txy[sl[k]];
            p23[k] = wb.tzq[sl[k]];
            const double dx = p01[k].x - xs, dy = p01[k].y - ys, dz = p23[k].x - zs;
            u[k] = fma(dz, dz, fma(dy, dy, dx * dx));
            y[k] = rsqrt_nr(u[k]);
            tv[k] = fma(u[k], a.pscale, -1.0);
            p[k] = a.pc[DEG];
        }
#pragma unroll
        for (int i = DEG - 1; i >= 0; --i) {
#pragma unroll
            for (int k = 0; k < NT; ++k) p[k] = fma(p[k], tv[k], a.pc[i]);
        }
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            bool ok = below_bits(u[k], lim);
            if (OWN) ok = ok && ((vt >> (t + k)) & 1u);
            // 1/r > 1e14 (hi word): r < 1e-14, a coincidence (realspace.py:118-122)
            sing = sing || (ok && __double2hiint(y[k]) > 0x42D6BCC4);
            const double w = ok ? y[k] - p[k] : 0.0;
            double *slot = &wb.acc[0][sl[k]][lane];
            *slot = fma(qs, w, *slot);
            if (NEWTON) accs = fma(p23[k].y, w, accs);
        }
    }
    singular |= sing ? 1 : 0;
    if (NEWTON && lane < m) atomicAdd(acc_s + lane, accs);
    __syncwarp();
}

// Dense batch of the Newton field (DEG > 0: the polynomial pair factor
// g = w^2 (w - R(r^2)), hit_value_field_poly): the structure of
// dense_batch_poly with three components -- the target side E_t += q_s g d
// (d = x_t - x_s) into the lane-owned rows acc[c][slot][lane], the source
// side E_s -= q_t g d in registers, leaving with three REDG per source and
// batch instead of three per pair.
template <int DEG, bool OWN, class WB>
__device__ __forceinline__ void dense_batch_field_poly(WB &wb, int lane, int j, int m, double xs, double ys, double zs,
                                                       double qs, const RealArgs &a, unsigned amask, int tbase,
                                                       double *__restrict__ acc_s, int &singular) {
    constexpr int NT = SE_DENSE_NT;
    unsigned vt = 0xffffu;
    if (OWN) {
        const int c = min(max(j - tbase, 0), kT);
        vt = amask & ((1u << c) - 1u);
    }
    const long long lim = __double_as_longlong(a.rc2x);
    double ax = 0.0, ay = 0.0, az = 0.0;
    bool sing = false;
#pragma unroll 1
    for (int t = 0; t < kT; t += NT) {
        int sl[NT];
        double dx[NT], dy[NT], dz[NT], qt[NT], u[NT], y[NT], tv[NT], p[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            sl[k] = tslot(t + k);
            const double2 p01 = wb.txy[sl[k]], p23 = wb.tzq[sl[k]];
            dx[k] = p01.x - xs;
            dy[k] = p01.y - ys;
            dz[k] = p23.x - zs;
            qt[k] = p23.y;
            u[k] = fma(dz[k], dz[k], fma(dy[k], dy[k], dx[k] * dx[k]));
            y[k] = rsqrt_nr(u[k]);
            tv[k] = fma(u[k], a.pscale, -1.0);
            p[k] = a.pc[DEG];
        }
#pragma unroll
        for (int i = DEG - 1; i >= 0; --i) {
#pragma unroll
            for (int k = 0; k < NT; ++k) p[k] = fma(p[k], tv[k], a.pc[i]);
        }
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            bool ok = below_bits(u[k], lim);
            if (OWN) ok = ok && ((vt >> (t + k)) & 1u);
            sing = sing || (ok && __double2hiint(y[k]) > 0x42D6BCC4);  // r < 1e-14
            const double g = ok ? (y[k] * y[k]) * (y[k] - p[k]) : 0.0;
            const double gs = qs * g, gt = qt[k] * g;
            double *s0 = &wb.acc[0][sl[k]][lane], *s1 = &wb.acc[1][sl[k]][lane], *s2 = &wb.acc[2][sl[k]][lane];
            *s0 = fma(gs, dx[k], *s0);
            *s1 = fma(gs, dy[k], *s1);
            *s2 = fma(gs, dz[k], *s2);
            ax = fma(-gt, dx[k], ax);
            ay = fma(-gt, dy[k], ay);
            az = fma(-gt, dz[k], az);
        }
    }
    singular |= sing ? 1 : 0;
    if (lane < m) {
        atomicAdd(acc_s + 3 * lane, ax);
        atomicAdd(acc_s + 3 * lane + 1, ay);
        atomicAdd(acc_s + 3 * lane + 2, az);
    }
    __syncwarp();
}

// One batch of <= 32 candidate sources [jb, jb+m) of a neighbour-cell run:
//  1. fp32 prefilter of all 16 x m (target, source) pairs: lane l tests
//     targets (l % 8, l % 8 + 8) against sources 8 (l / 8) .. + 7, two tests
//     per packed instruction; hit bit 2 kk + h = (target pa + 8 h, source
//     8 (l / 8) + kk).  Outside minimum-image mode the test is
//     |t'|^2 + |s'|^2 - 2 t'.s' - bound < 0 with t', s' relative to the
//     unit's origin; the bound covers the fp32 rounding.  With NEWTON,
//     sources of the target's own column count only if j > t;
//  2. warp prefix scan of the hit counts and compaction of the hits;
//  3. the list is evaluated 64 hits at a time (two per lane) on full warps.
template <bool MI, bool COUNT, bool NEWTON, bool WIDE, bool FLD, int DEGP>
__device__ __forceinline__ void pair_batch(const double4 *__restrict__ rec, int jb, int j1, double shx, double shy,
                                           double shz, const RealArgs &a, WarpBufT<FLD> &wb, int lane,
                                           const PreTargets &pt, const double3 org, int tbase, int hs,
                                           double *__restrict__ acc_src, int &singular, long long &cnt) {
    // polynomial pair term: DEG for the Newton potential, DEGF for the field
    constexpr int DEG = FLD ? 0 : DEGP, DEGF = FLD ? DEGP : 0;
    const int j = jb + lane;
    // the lane's own source stays in registers for the dense path (zero
    // past the end of the run: finite, never evaluated)
    const double far = -(8.0 * a.L + 4.0 * a.rc);  // past the end: r > rc from every target
    double xs = far, ys = far, zs = far, qs = 0.0;
    if (j < j1) {
        const double4 r = rec[j];
        if (j + 32 < j1) prefetch_l1(rec + j + 32);  // the run's next batch
        xs = r.x + shx;
        ys = r.y + shy;
        zs = r.z + shz;
        qs = r.w;
        wb.sxy[lane] = make_double2(xs, ys);
        wb.szq[lane] = make_double2(zs, r.w);
        if (MI) {
            wb.sf[lane] = make_float4((float)xs, (float)ys, (float)zs, 0.f);
        } else {
            const float fx = (float)(xs - org.x), fy = (float)(ys - org.y), fz = (float)(zs - org.z);
            wb.sf[lane] = make_float4(fx, fy, fz, fmaf(fz, fz, fmaf(fy, fy, fx * fx)));
        }
    }
    __syncwarp();
    const int m = min(32, j1 - jb);
    const int g8 = (lane >> 3) << 3;  // first source of this lane's quarter
    unsigned hit = 0;
    if (MI) {
        const float ax = __uint_as_float((unsigned)pt.x), bx = __uint_as_float((unsigned)(pt.x >> 32));
        const float ay = __uint_as_float((unsigned)pt.y), by = __uint_as_float((unsigned)(pt.y >> 32));
        const float az = __uint_as_float((unsigned)pt.z), bz = __uint_as_float((unsigned)(pt.z >> 32));
        const float aw = __uint_as_float((unsigned)pt.w), bw = __uint_as_float((unsigned)(pt.w >> 32));
        auto test = [&](float tx, float ty, float tz, float tw, const float4 p) -> unsigned {
            float dx = tx - p.x, dy = ty - p.y, dz = tz - p.z;
            if (a.mode[0] == 2) dx = min_image_f(dx, a.Lf, a.invLf);
            if (a.mode[1] == 2) dy = min_image_f(dy, a.Lf, a.invLf);
            if (a.mode[2] == 2) dz = min_image_f(dz, a.Lf, a.invLf);
            return fmaf(dz, dz, fmaf(dy, dy, dx * dx)) < a.rc2f + tw ? 1u : 0u;  // tw: 0 or +inf-like
        };
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const float4 p = wb.sf[g8 + kk];
            hit |= test(ax, ay, az, aw, p) << (2 * kk);
            hit |= test(bx, by, bz, bw, p) << (2 * kk + 1);
        }
    } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const float4 p = wb.sf[g8 + kk];
            const unsigned long long d = f2fma(pt.x, p.x, f2fma(pt.y, p.y, f2fma(pt.z, p.z, f2add(pt.w, p.w))));
            // sign bits of the two results -> bits 2 kk (target a), 2 kk + 1 (b)
            hit |= (((unsigned)d >> 31) | (((unsigned)(d >> 32) >> 30) & 2u)) << (2 * kk);
        }
    }
    if (m < 32) {  // sources past the end of the run
        const int valid = min(max(m - g8, 0), 8);
        hit &= valid >= 8 ? 0xffffu : ((1u << (2 * valid)) - 1u);
    }
    if (NEWTON && hs >= 0) {
        // own-column sources j in [hs, t] are visited from their own unit:
        // exclude source slots k in [lo, t - jb] for each of the two targets
        const int lo = max(hs - jb, 0) - g8;
        auto excl = [&](int t) -> unsigned {  // 8-bit mask over this quarter
            const int hi = t - jb - g8;
            const int l0 = max(lo, 0), h0 = min(hi, 7);
            if (h0 < l0) return 0u;
            return ((2u << h0) - 1u) & ~((1u << l0) - 1u);
        };
        auto spread = [](unsigned x) {  // bit i -> bit 2 i
            x = (x | (x << 4)) & 0x0f0fu;
            x = (x | (x << 2)) & 0x3333u;
            return (x | (x << 1)) & 0x5555u;
        };
        hit &= ~(spread(excl(tbase + pt.ta)) | (spread(excl(tbase + pt.tb)) << 1));
    }
    const int c = __popc(hit);
    if (!COUNT && (FLD ? (NEWTON && DEGF > 0) : (NEWTON || DEG > 0)) &&
        __reduce_add_sync(0xffffffffu, (unsigned)c) >= (unsigned)a.dense_min) {
        if constexpr (!NEWTON && !FLD) {
            // full shell (deterministic mode): every batch may hold the unit's own
            // targets as sources; the self pair is dropped by its index
            dense_batch_poly<(DEG > 0 ? DEG : 1), true, false>(wb, lane, j, m, xs, ys, zs, qs, a, pt.amask, tbase,
                                                               nullptr, singular);
        } else if constexpr (FLD) {
            constexpr int DF = DEGF > 0 ? DEGF : 1;
            if (hs >= 0)
                dense_batch_field_poly<DF, true>(wb, lane, j, m, xs, ys, zs, qs, a, pt.amask, tbase, acc_src + 3 * jb,
                                                 singular);
            else
                dense_batch_field_poly<DF, false>(wb, lane, j, m, xs, ys, zs, qs, a, pt.amask, tbase, acc_src + 3 * jb,
                                                  singular);
        } else if (DEG > 0) {
            if (hs >= 0)
                dense_batch_poly<DEG, true>(wb, lane, j, m, xs, ys, zs, qs, a, pt.amask, tbase, acc_src + jb, singular);
            else
                dense_batch_poly<DEG, false>(wb, lane, j, m, xs, ys, zs, qs, a, pt.amask, tbase, acc_src + jb,
                                             singular);
        } else
            dense_batch<WIDE>(wb, lane, j, m, xs, ys, zs, qs, a, pt.amask, tbase, hs, org, acc_src + jb, singular);
        return;
    }
    const int incl = warp_incl_scan(c, lane);
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int pos = incl - c;
    {   // fixed, fully predicated compaction of this lane's <= 16 hit bits
        unsigned taga, tagb;  // pinned in registers (not rematerialised per bit)
        asm volatile("mov.b32 %0, %1;" : "=r"(taga) : "r"(((unsigned)tslot(pt.ta) << 5) | (unsigned)g8));
        asm volatile("mov.b32 %0, %1;" : "=r"(tagb) : "r"(((unsigned)tslot(pt.tb) << 5) | (unsigned)g8));
        unsigned short *dst = wb.ent + pos;
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (hit & (1u << b)) *dst++ = (unsigned short)(((b & 1) ? tagb : taga) + (b >> 1));
    }
    __syncwarp();
    double *__restrict__ acc_batch = acc_src + (FLD ? 3 : 1) * jb;  // source-side sums of this batch
    for (int e0 = 0; e0 < total; e0 += 64) {
        const int rem = total - e0;
        if (rem > 32) {
            // two hits per lane in one basic block (the second one a masked
            // duplicate of the first on lanes past the end of the list)
            const bool v2 = lane < rem - 32;
            const unsigned en1 = wb.ent[e0 + lane];
            const unsigned en2 = v2 ? wb.ent[e0 + 32 + lane] : en1;
            Hit h1, h2;
            if (DEG > 0) {
                hit_poly<(DEG > 0 ? DEG : 1), NEWTON>(en1, true, a, wb, singular, h1, jb, tbase);
                hit_poly<(DEG > 0 ? DEG : 1), NEWTON>(en2, v2, a, wb, singular, h2, jb, tbase);
            } else {
                const double x1 = hit_geometry<MI, NEWTON, FLD>(en1, true, a, wb, jb, tbase, singular, h1);
                const double x2 = hit_geometry<MI, NEWTON, FLD>(en2, v2, a, wb, jb, tbase, singular, h2);
                if (FLD && DEGF > 0) {
                    hit_value_field_poly<(DEGF > 0 ? DEGF : 1)>(a, h1);
                    hit_value_field_poly<(DEGF > 0 ? DEGF : 1)>(a, h2);
                } else {
                    hit_value<WIDE, FLD>(x1, a, h1);
                    hit_value<WIDE, FLD>(x2, a, h2);
                }
            }
            if (COUNT) {
                cnt += (h1.ok ? (NEWTON ? 2 : 1) : 0) + (h2.ok ? (NEWTON ? 2 : 1) : 0);
            } else {
                apply_hit<NEWTON, FLD>(h1, wb, lane, acc_batch);
                apply_hit<NEWTON, FLD>(h2, wb, lane, acc_batch);
            }
        } else if (lane < rem) {
            Hit h;
            if (DEG > 0) {
                hit_poly<(DEG > 0 ? DEG : 1), NEWTON>(wb.ent[e0 + lane], true, a, wb, singular, h, jb, tbase);
            } else if (FLD && DEGF > 0) {
                hit_geometry<MI, NEWTON, FLD>(wb.ent[e0 + lane], true, a, wb, jb, tbase, singular, h);
                hit_value_field_poly<(DEGF > 0 ? DEGF : 1)>(a, h);
            } else {
                h = eval_hit<MI, NEWTON, WIDE, FLD>(wb.ent[e0 + lane], a, wb, jb, tbase, singular);
            }
            if (COUNT)
                cnt += h.ok ? (NEWTON ? 2 : 1) : 0;
            else
                apply_hit<NEWTON, FLD>(h, wb, lane, acc_batch);
        }
    }
    __syncwarp();
}

// First index j in [lo, hi) with
// Q(z_j) >= qt (upper: > qt), or hi, by bisection.
__device__ __forceinline__ int zbound(const double4 *__restrict__ rec, int lo, int hi, int qt, bool upper,
                                      double qinv) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int qz = zq(__ldg(&rec[mid].z), qinv);
        if (upper ? qz > qt : qz >= qt)
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

// NEWTON: every unordered pair once -- neighbour cells in the half shell
// (ox, oy) > 0 (lexicographic) plus own-column pairs with t < j; the
// partial sums of both sides go to acc_src (sorted order, zeroed before) and
// a finishing kernel scatters them.  Otherwise the full column neighbourhood
// and direct writes of phi (minimum-image mode for < 5 cells per axis).
template <bool MI, bool COUNT, bool NEWTON, bool WIDE, bool FLD, int DEG = 0>
__global__ void __launch_bounds__(32 * kWarps, FLD ? kMinBlocksField : kMinBlocks) realspace_cell_kernel(
    const double4 *__restrict__ rec, const int *__restrict__ sidx, const int *__restrict__ starts,
    const int4 *__restrict__ units, const int *__restrict__ nunits, RealArgs a, double *__restrict__ phi,
    double *__restrict__ acc_src, int *__restrict__ flag, unsigned long long *__restrict__ npairs) {
    static_assert(DEG == 0 || (!MI && !COUNT && !WIDE), "polynomial pair term: cell path, narrow erfc range");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpBufT<FLD> &wb = reinterpret_cast<WarpBufT<FLD> *>(smem_raw)[warp];
    // units from the one holding this shard's first target (nunits[1]; 0 for
    // one rank): a rank launches only about its share of the units
    const int u = nunits[1] + blockIdx.x * kWarps + warp;
    if (u >= *nunits) return;
    const int4 un = units[u];
    const int n = a.n;
    const int col = un.x;  // bins are columns (cx, cy) of edge >= rc/3, sorted by z inside
    const int cx = col / n, cy = col - cx * n;
    const int tl = lane & (kT - 1);
    const int t = un.y + tl;
    const bool active = tl < un.z && t >= a.rlo && t < a.rhi;
    if (__ballot_sync(0xffffffffu, active) == 0) return;
    // inactive slots far away (r > rc from every source; dense_batch_poly)
    const double farT = 8.0 * a.L + 4.0 * a.rc;
    const double4 tp = active ? rec[t] : make_double4(farT, farT, farT, 0);
    if (lane < kT) {
        wb.txy[tslot(lane)] = make_double2(tp.x, tp.y);
        wb.tzq[tslot(lane)] = make_double2(tp.z, tp.w);
    }
#pragma unroll
    for (int c = 0; c < (FLD ? 3 : 1); ++c)
        for (int i = 0; i < kT; ++i) wb.acc[c][i][lane] = 0.0;
    // z extent of the unit's targets (a unit is a z-slab of its column)
    double zmin = active ? tp.z : 1e300, zmax = active ? tp.z : -1e300;
    for (int o = 16; o > 0; o >>= 1) {
        zmin = fmin(zmin, __shfl_xor_sync(0xffffffffu, zmin, o));
        zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    }
    __syncwarp();
    // prefilter operands of this lane's two targets (see PreTargets), relative
    // to org = (column corner, zmin); the fp32 rounding margin of the expanded
    // form scales with the operand magnitudes: |t'| <= Rt, |s'| <= Rt + rc
    const double3 org = make_double3(cx * a.edge, cy * a.edge, zmin);
    if (lane < kT)
        wb.tf[lane] = make_float4((float)(tp.x - org.x), (float)(tp.y - org.y), (float)(tp.z - org.z), active ? 0.f : 1.f);
    __syncwarp();
    PreTargets pt;
    {
        const double Rt = 1.4143 * a.edge + (zmax - zmin), Rs = Rt + 1.01 * a.rc;
        const float bound = (float)(a.rc2 + 4e-7 * (Rt + Rs) * (Rt + Rs));
        const unsigned amask = __ballot_sync(0xffffffffu, active);
        pt.amask = amask;
        pt.ta = lane & 7;
        pt.tb = pt.ta + 8;
        float v[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int sl = h ? pt.tb : pt.ta;
            const double4 q = make_double4(wb.txy[tslot(sl)].x, wb.txy[tslot(sl)].y, wb.tzq[tslot(sl)].x, 0.0);
            const bool ok = (amask >> sl) & 1u;
            if (MI) {
                v[h][0] = (float)q.x;
                v[h][1] = (float)q.y;
                v[h][2] = (float)q.z;
                v[h][3] = ok ? 0.f : -1e30f;
            } else {
                const float rx = (float)(q.x - org.x), ry = (float)(q.y - org.y), rz = (float)(q.z - org.z);
                v[h][0] = -2.f * rx;
                v[h][1] = -2.f * ry;
                v[h][2] = -2.f * rz;
                v[h][3] = ok ? fmaf(rz, rz, fmaf(ry, ry, rx * rx)) - bound : 1e30f;
            }
        }
        pt.x = f2pack(v[0][0], v[1][0]);
        pt.y = f2pack(v[0][1], v[1][1]);
        pt.z = f2pack(v[0][2], v[1][2]);
        pt.w = f2pack(v[0][3], v[1][3]);
    }
    int singular = 0;
    long long cnt = 0;

    auto run = [&](int j0, int j1, double shx, double shy, double shz, int hs) {
        for (int jb = j0; jb < j1; jb += 32)
            pair_batch<MI, COUNT, NEWTON, WIDE, FLD, DEG>(rec, jb, j1, shx, shy, shz, a, wb, lane, pt, org, un.y, hs, acc_src,
                                                singular, cnt);
    };
    if (MI) {
        // every column once, the whole column, minimum image in the distance
        for (int xc = 0; xc < n; ++xc)
            for (int yc = 0; yc < n; ++yc) {
                const int cs = starts[xc * n + yc], ce = starts[xc * n + yc + 1];
                if (cs < ce) run(cs, ce, 0.0, 0.0, 0.0, -1);
            }
    } else {
        // The half shell's columns, one per lane (<= 25 for reach 3): own
        // row (ox = cx, oy = cy .. cy + R), then rows ox = cx + 1 .. cx + R
        // (oy = cy - R .. cy + R).  Each lane locates its column's runs by a
        // scalar binary search, all columns concurrently (the searches were
        // a chain of dependent L2 loads per column).  Sources with
        // |z_s - z_t| <= h, h^2 = rc^2 - (lateral gap)^2, for some target can
        // be within rc (one quantum of slack each side):
        //   [j0, j1)  in-box window (own column: sources above the unit, j > t)
        //   [k0, ce)  the window's part below z = 0, as the image shifted by -L
        //   [cs, k1)  its part above z = L, shifted by +L (periodic z only)
        // NEWTON: the half shell ((R + 1) + R (2R + 1) columns); otherwise
        // (the deterministic mode) the full shell of (2R + 1)^2 columns,
        // R = 2: <= 25 lanes, each target summing all its partners itself
        const int R = a.reach, nc = NEWTON ? (R + 1) + R * (2 * R + 1) : (2 * R + 1) * (2 * R + 1);
        int j0 = 0, j1 = 0, k0 = 0, k1 = 0, cs = 0, ce = 0, shc = 0;  // shc: x, y image codes (-1, 0, 1)
        if (lane < nc) {
            int ox, oy;
            if (!NEWTON) {
                ox = cx - R + lane / (2 * R + 1);
                oy = cy - R + lane % (2 * R + 1);
            } else if (lane <= R) {
                ox = cx;
                oy = cy + lane;
            } else {
                const int i = lane - R - 1;
                ox = cx + 1 + i / (2 * R + 1);
                oy = cy - R + i % (2 * R + 1);
            }
            int xc = ox, yc = oy, sx = 0, sy = 0;
            bool ok = true;
            if (a.mode[0] == 1) {
                if (xc < 0) { xc += n; sx = -1; }
                else if (xc >= n) { xc -= n; sx = 1; }
            } else {
                ok = ok && xc >= 0 && xc < n;
            }
            if (a.mode[1] == 1) {
                if (yc < 0) { yc += n; sy = -1; }
                else if (yc >= n) { yc -= n; sy = 1; }
            } else {
                ok = ok && yc >= 0 && yc < n;
            }
            // the z-window: sources within rc of some target t satisfy
            // |z_s - z_t| <= h_t, h_t^2 = rc^2 - (lateral distance from t to
            // the source column's cell)^2 -- per target (the unit's targets
            // spread over their own column's cross-section: ~10% fewer
            // candidates than one window from the two cells' gap)
            // (fp32 relative to the unit origin; h_t from h_t^2 + eps2, eps2 =
            // 4e-6 rc^2 above the fp32 error of h_t^2, and 1e-5 rc more on
            // each side: a superset of the exact window)
            double wlo = 1e300, whi = -1e300;
            if (ok) {
                const float x0 = (float)((ox - cx) * a.edge), y0 = (float)((oy - cy) * a.edge), e = (float)a.edge;
                const float rc2f = (float)a.rc2, eps2 = 4e-6f * rc2f;
                float lo = 3e38f, hi = -3e38f;
                for (int tt = 0; tt < kT; ++tt) {
                    const float4 q = wb.tf[tt];
                    const float gxt = fmaxf(0.f, fmaxf(x0 - q.x, q.x - (x0 + e)));
                    const float gyt = fmaxf(0.f, fmaxf(y0 - q.y, q.y - (y0 + e)));
                    const float h2t = rc2f - gxt * gxt - gyt * gyt;
                    if (q.w == 0.f && h2t >= -eps2) {
                        const float ht = sqrtf(h2t + eps2);
                        lo = fminf(lo, q.z - ht);
                        hi = fmaxf(hi, q.z + ht);
                    }
                }
                ok = lo <= hi;
                wlo = org.z + (double)lo - 1e-5 * a.rc;
                whi = org.z + (double)hi + 1e-5 * a.rc;
            }
            if (ok) {
                cs = starts[xc * n + yc];
                ce = starts[xc * n + yc + 1];
                const bool own = NEWTON && lane == 0;  // own column: sources above the unit only
                j0 = own ? un.y + 1 : zbound(rec, cs, ce, zq(wlo, a.qinv) - 1, false, a.qinv);
                j1 = zbound(rec, j0, ce, zq(whi, a.qinv) + 1, true, a.qinv);
                k0 = ce;
                k1 = cs;
                if (a.zper) {
                    if (!own && wlo < 0.0) k0 = zbound(rec, cs, ce, zq(wlo + a.L, a.qinv) - 1, false, a.qinv);
                    if (whi >= a.L) k1 = zbound(rec, cs, ce, zq(whi - a.L, a.qinv) + 1, true, a.qinv);
                }
                shc = (sx + 1) * 3 + (sy + 1);
            }
        }
        for (int c = 0; c < nc; ++c) {
            const int c0 = __shfl_sync(0xffffffffu, j0, c), c1 = __shfl_sync(0xffffffffu, j1, c);
            const int ck0 = __shfl_sync(0xffffffffu, k0, c), cce = __shfl_sync(0xffffffffu, ce, c);
            const int ccs = __shfl_sync(0xffffffffu, cs, c), ck1 = __shfl_sync(0xffffffffu, k1, c);
            const int code = __shfl_sync(0xffffffffu, shc, c);
            {   // the next column's first batch
                const int n0 = __shfl_sync(0xffffffffu, j0, (c + 1) & 31), n1 = __shfl_sync(0xffffffffu, j1, (c + 1) & 31);
                if (c + 1 < nc && n0 + lane < n1) prefetch_l1(rec + n0 + lane);
            }
            const double shx = (code / 3 - 1) * a.L, shy = (code % 3 - 1) * a.L;
            if (c0 < c1) run(c0, c1, shx, shy, 0.0, (NEWTON && c == 0) ? un.y : -1);
            if (ck0 < cce) run(ck0, cce, shx, shy, -a.L, -1);
            if (ccs < ck1) run(ccs, ck1, shx, shy, a.L, -1);
        }
    }
    if (COUNT) {
        long long c = cnt;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) atomicAdd(npairs, (unsigned long long)c);
        return;
    }
    if (__any_sync(0xffffffffu, singular) && lane == 0) atomicExch(flag, 1);
    __syncwarp();
    if (active && lane < kT) {
#pragma unroll
        for (int c = 0; c < (FLD ? 3 : 1); ++c) {
            double v = 0.0;
            for (int i = 0; i < 32; ++i) v += wb.acc[c][tslot(tl)][(tl + i) & 31];
            if (FLD) {
                // field: no self term (the Ewald self-interaction is a constant)
                if (NEWTON)
                    atomicAdd(acc_src + 3 * t + c, v);
                else
                    phi[3 * (int64_t)sidx[t] + c] = v;
            } else if (NEWTON) {
                atomicAdd(acc_src + t, v);
            } else {
                if (a.add_self) v += (-2.0 * a.xi * tp.w) / a.sqrtpi;
                phi[sidx[t]] = v;
            }
        }
    }
}

// NEWTON finish, field mode: E[orig] = accumulated (3 components)
__global__ void realspace_finish_field_kernel(const double *__restrict__ acc, const int *__restrict__ sidx, int64_t N,
                                              double *__restrict__ E) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t o = 3 * (int64_t)sidx[i];
    E[o] = acc[3 * i];
    E[o + 1] = acc[3 * i + 1];
    E[o + 2] = acc[3 * i + 2];
}

// NEWTON finish: phi[orig] = accumulated pair sums (+ the self term of owned targets)
__global__ void realspace_finish_kernel(const double *__restrict__ acc, const double4 *__restrict__ rec,
                                        const int *__restrict__ sidx, int64_t N, RealArgs a, double *__restrict__ phi) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    double v = acc[i];
    const int o = sidx[i];
    if (a.add_self && (a.n_own >= 0 ? o < a.n_own : (i >= a.rlo && i < a.rhi))) v += (-2.0 * a.xi * rec[i].w) / a.sqrtpi;
    phi[o] = v;
}

// rc > L/2 with periodic axes: explicit images (realspace.py:138-165)
template <bool FLD>
__global__ void realspace_image_kernel(const double *__restrict__ pos, const double *__restrict__ q, int64_t N,
                                       int64_t rlo, int64_t rhi, RealArgs a, int D, int layers,
                                       double *__restrict__ phi, int *__restrict__ flag) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N) return;
    bool own = t >= rlo && t < rhi;
    if (!own) return;
    double xt = pos[3 * t], yt = pos[3 * t + 1], zt = pos[3 * t + 2];
    int lx = D >= 1 ? layers : 0, ly = D >= 2 ? layers : 0, lz = D >= 3 ? layers : 0;
    double acc = 0.0, ex = 0.0, ey = 0.0, ez = 0.0;
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
                    if (r < a.rc) {
                        if (FLD) {
                            const double g = q[s] * (erfc(a.xi * r) / r + kTwoOverSqrtPi * a.xi * exp(-a.xi * a.xi * r * r)) / (r * r);
                            ex += g * dx;
                            ey += g * dy;
                            ez += g * dz;
                        } else {
                            img += q[s] * (erfc(a.xi * r) / r);
                        }
                    }
                }
                acc += img;
            }
    if (err) atomicMax(flag, err);
    if (FLD) {
        phi[3 * t] = ex;
        phi[3 * t + 1] = ey;
        phi[3 * t + 2] = ez;
        return;
    }
    double v = acc;
    if (a.add_self) v += (-2.0 * a.xi * q[t]) / a.sqrtpi;
    phi[t] = v;
}

// The polynomial pair term (pair_poly) for this xi, rc: coefficients and
// degree by pair_poly_fit (se_host.cpp, long double); 0 (erfc_fast) when no
// degree <= 32 reaches the accuracy (xi rc > ~5) or SE_B200_PAIR_POLY=0.
static int fit_pair_poly(se_plan *pl, RealArgs &a, int kind) {
    a.rc2x = a.rc * a.rc;
    a.pscale = 2.0 / a.rc2x;
    static const bool off = [] {
        const char *e = std::getenv("SE_B200_PAIR_POLY");
        return e && std::atoi(e) == 0;
    }();
    if (off) {
        a.pdeg = 0;
        return 0;
    }
    se_plan::PairPoly &c = pl->pair_poly[kind];  // fitted once per plan (the fit is ~1 ms of host work)
    if (!c.valid || c.xi != a.xi || c.rc != a.rc) {
        c.deg = pair_poly_fit(a.xi, a.rc, kind, c.pc);
        c.xi = a.xi;
        c.rc = a.rc;
        c.valid = true;
    }
    for (int i = 0; i < 33; ++i) a.pc[i] = c.pc[i];
    a.pdeg = c.deg;
    return a.pdeg;
}

// Prefilter hits (of kT x 32 slots) from which a batch is evaluated densely
// (dense_batch).  SE_B200_DENSE_MIN overrides it (A/B runs; > 512 disables).
static int dense_threshold() {
    static const int v = [] {
        const char *e = std::getenv("SE_B200_DENSE_MIN");
        return e ? std::atoi(e) : kDenseMin;
    }();
    return v;
}

// targets per work unit: kT, or half of it for small systems (latency bound:
// more, shorter units keep more warps in flight)
// (by the total particle count: for a shard of a large system the 16-target
// units stay faster -- 8-target units measured 2.27 vs 1.96 ms per cfg2 rank
// at 8 ranks)
static int real_unit(int64_t N) { return N < 50000 ? kT / 2 : kT; }

// columns of edge >= rc/reach and the particle binning by (column, z)
static void cell_bin(se_plan *pl, const double *pos, const double *q, int64_t N, RealArgs &a, bool full = false) {
    const double L = pl->L, rc = pl->p.rc;
    if (N >= (1LL << 27)) fail(SE_EINVAL, "real-space kernel supports N < 2^27 particles per call");
    CellGeom &c = pl->cell;
    // columns (cx, cy) of edge >= rc/reach in x, y; z is not binned but sorted
    int reach = kReachMax;
    long long nn = 1;
    if (pl->dom.ncols > 0) {
        // domain mode: the caller's column grid (identical on every rank)
        nn = pl->dom.ncols;
        reach = (int)std::ceil(rc * (double)nn / L - 1e-12);
        if (reach < 1) reach = 1;
        if (reach > kReachMax || nn > 1024)
            fail(SE_EINVAL, "domain column grid: columns must be at least rc / 3 wide and at most 1024 per axis");
    } else {
        if (full) reach = 2;  // the full shell must fit one lane per column
        for (;; --reach) {
            nn = (long long)std::floor(reach * L / rc);
            if (nn < 1) nn = 1;
            if (nn > 1024) nn = 1024;
            if (reach == 2 || (double)N / ((double)nn * nn) >= kShortColumn) break;
        }
    }
    a.reach = reach;
    c.n = (int)nn;
    c.edge = L / c.n;
    // x, y: periodic axes wrap +-reach columns if there are enough of them,
    // else all columns with the minimum image (then z too, if periodic)
    for (int ax = 0; ax < 2; ++ax) c.mode[ax] = ax < pl->D ? (c.n >= 2 * reach + 1 ? 1 : 2) : 0;
    const bool mi = c.mode[0] == 2 || c.mode[1] == 2;
    if (pl->dom.ncols > 0 && mi)
        fail(SE_EINVAL, "domain mode needs at least 2 reach + 1 columns per periodic axis (no minimum-image mode)");
    c.mode[2] = pl->D == 3 ? (mi ? 2 : 1) : 0;
    a.n = c.n;
    a.edge = c.edge;
    a.zper = c.mode[2] == 1;
    int nbins = c.n * c.n;
    {
        // z quantum L / 2^kb <= rc / 256 at least: the windows' one-quantum
        // slack costs nothing measurable.  The counting sort's fine bins
        // (column, quantum) stay <= max(2^22, 4 N) (cfg2: 900 columns x 2^12
        // quanta; a coarser quantum would only widen the windows' slack)
        int cb = 1;
        while ((1LL << cb) < (long long)nbins) ++cb;
        int kz = 8;
        while (kz < 20 && (double)(1 << kz) < 256.0 * L / rc) ++kz;
        // as fine as the counting sort's bin budget allows (clustered inputs
        // then keep ~1 particle per fine bin as well)
        const long long fine_cap = std::max<long long>(1LL << 22, 4LL * N);
        a.kb = std::max(kz, 1);
        while (a.kb < 20 && ((long long)nbins << (a.kb + 1)) <= fine_cap) ++a.kb;
        a.kb = std::min(32 - cb, a.kb);
        while (a.kb > 1 && ((long long)nbins << a.kb) > fine_cap) --a.kb;
        a.qinv = (double)(1 << a.kb) / L;
    }
    for (int ax = 0; ax < 3; ++ax) a.mode[ax] = c.mode[ax];
    cudaStream_t st = pl->stream;
    prof_begin(pl, SE_K_SORT);
    const int unit = real_unit(N);
    binning_reserve(pl, pl->cbin, N, nbins, unit, a.kb);
    SE_CUDA(cudaMemsetAsync(pl->cbin.counts.ptr, 0, sizeof(int) * (nbins + 1), st));
    if (nbins <= kHistSmem) {
        int64_t blocks = (N + 4095) / 4096;  // ~16 particles per thread
        if (blocks > 1184) blocks = 1184;
        cell_keys_hist_kernel<<<(unsigned)blocks, 256, sizeof(int) * nbins, st>>>(
            pos, N, a, nbins, pl->cbin.keys.as<unsigned>(), pl->cbin.counts.as<int>());
    } else {
        cell_keys_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(pos, N, a, pl->cbin.keys.as<unsigned>(),
                                                                       pl->cbin.counts.as<int>());
    }
    SE_LAUNCH_CHECK();
    pl->launches += 1;
    if (pl->dom.ncols > 0)  // units (targets) only in the own columns cx in [col_lo, col_hi)
        binning_sort(pl, pl->cbin, pos, q, N, nbins, unit, a.kb, -1, pl->dom.col_lo * c.n, pl->dom.col_hi * c.n);
    else
        binning_sort(pl, pl->cbin, pos, q, N, nbins, unit, a.kb, a.rlo);
    prof_end(pl, SE_K_SORT);
}

// The full shell without Newton's third law: in the deterministic mode (no
// source-side atomics), and for the field when its polynomial pair factor is
// not available -- all of the erfc-path field's pairs go through the
// compacted path with three source-side fp64 atomics each, which costs more
// than evaluating every pair twice (cfg2: 30.5 ms full shell against 33.9 ms
// with Newton).  With the polynomial factor the field runs the half shell
// with Newton like the potential: its dense batches keep the source side in
// registers (three REDG per source and batch, dense_batch_field_poly).
// (the domain decomposition relies on the +x half shell: Newton there)
static bool narrow_erfc(const RealArgs &a) { return !(a.xi * a.rc * (1.0 + 1e-4) > SE_ERFC_XMAX); }
template <bool FLD>
static bool full_shell(const se_plan *pl, const RealArgs &a) {
    if (pl->dom.ncols != 0) return false;
    if (pl->deterministic) return true;
    static const bool newton_field = [] {
        const char *e = std::getenv("SE_B200_FIELD_NEWTON");  // A/B: 0 = the full-shell field
        return !(e && std::atoi(e) == 0);
    }();
    return FLD && !(newton_field && a.pdeg > 0 && narrow_erfc(a));
}

template <bool COUNT, bool FLD = false>
static void launch_cell(se_plan *pl, int64_t N, const RealArgs &a, double *phi, unsigned long long *npairs) {
    const CellGeom &c = pl->cell;
    int nbins = c.n * c.n;
    const int unit = real_unit(N);
    int64_t maxu = binning_max_units(pl->cbin, N, nbins, unit);
    // a shard [rlo, rhi) spans at most its targets / unit + one partial unit
    // per column + 1 units from nunits[1] on
    if (a.rhi - a.rlo < N) maxu = std::min<int64_t>(maxu, (a.rhi - a.rlo) / unit + nbins + 2);
    const bool mi = c.mode[0] == 2 || c.mode[1] == 2 || c.mode[2] == 2;
    // deterministic mode: no Newton (no source-side atomics), each target
    // sums its own partners in a fixed order
    const bool full = mi || full_shell<FLD>(pl, a);
    unsigned blocks = (unsigned)((maxu + kWarps - 1) / kWarps);
    cudaStream_t st = pl->stream;
    const size_t smem = sizeof(WarpBufT<FLD>) * kWarps;
    const int nc = FLD ? 3 : 1;
    double *acc = nullptr;
    if (!full) {
        pl->racc.ensure(sizeof(double) * nc * N);
        acc = pl->racc.as<double>();
        SE_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * nc * N, st));
    }
    auto args = [&](auto kern) {
        SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<blocks, 32 * kWarps, smem, st>>>(pl->cbin.rec.as<double4>(), pl->cbin.idx_sorted.as<int>(),
                                                pl->cbin.starts.as<int>(), pl->cbin.units.as<int4>(),
                                                pl->cbin.nunits.as<int>(), a, phi, acc, pl->flag.as<int>(), npairs);
    };
    if (!COUNT) prof_begin(pl, SE_K_REALSPACE);
    // narrow kernels: x = xi r <= xi rc (1 + 2e-5) for every prefiltered pair
    const bool wide = a.xi * a.rc * (1.0 + 1e-4) > SE_ERFC_XMAX;
    if (mi)
        args(wide ? realspace_cell_kernel<true, COUNT, false, true, FLD>
                  : realspace_cell_kernel<true, COUNT, false, false, FLD>);
    else if (full) {
        if constexpr (FLD && !COUNT) {
            switch (wide || pl->deterministic ? 0 : a.pdeg) {
                case 20: args(realspace_cell_kernel<false, false, false, false, true, 20>); break;
                case 24: args(realspace_cell_kernel<false, false, false, false, true, 24>); break;
                case 28: args(realspace_cell_kernel<false, false, false, false, true, 28>); break;
                case 32: args(realspace_cell_kernel<false, false, false, false, true, 32>); break;
                default:
                    args(wide ? realspace_cell_kernel<false, false, false, true, true>
                              : realspace_cell_kernel<false, false, false, false, true>);
            }
        } else if constexpr (!FLD && !COUNT) {
            // the deterministic potential: polynomial pair term and dense batches too
            switch (wide ? 0 : a.pdeg) {
                case 20: args(realspace_cell_kernel<false, false, false, false, false, 20>); break;
                case 24: args(realspace_cell_kernel<false, false, false, false, false, 24>); break;
                case 28: args(realspace_cell_kernel<false, false, false, false, false, 28>); break;
                case 32: args(realspace_cell_kernel<false, false, false, false, false, 32>); break;
                default:
                    args(wide ? realspace_cell_kernel<false, false, false, true, false>
                              : realspace_cell_kernel<false, false, false, false, false>);
            }
        } else {
            args(wide ? realspace_cell_kernel<false, COUNT, false, true, FLD>
                      : realspace_cell_kernel<false, COUNT, false, false, FLD>);
        }
    }
    else if constexpr (!COUNT && !FLD) {
        // the polynomial pair term where it is fitted (pair_poly)
        switch (wide ? 0 : a.pdeg) {
            case 20: args(realspace_cell_kernel<false, false, true, false, false, 20>); break;
            case 24: args(realspace_cell_kernel<false, false, true, false, false, 24>); break;
            case 28: args(realspace_cell_kernel<false, false, true, false, false, 28>); break;
            case 32: args(realspace_cell_kernel<false, false, true, false, false, 32>); break;
            default:
                args(wide ? realspace_cell_kernel<false, false, true, true, false>
                          : realspace_cell_kernel<false, false, true, false, false>);
        }
    } else if constexpr (!COUNT && FLD) {
        // the Newton field: only with the polynomial pair factor (full_shell)
        switch (wide ? 0 : a.pdeg) {
            case 20: args(realspace_cell_kernel<false, false, true, false, true, 20>); break;
            case 24: args(realspace_cell_kernel<false, false, true, false, true, 24>); break;
            case 28: args(realspace_cell_kernel<false, false, true, false, true, 28>); break;
            case 32: args(realspace_cell_kernel<false, false, true, false, true, 32>); break;
            default:
                args(wide ? realspace_cell_kernel<false, false, true, true, true>
                          : realspace_cell_kernel<false, false, true, false, true>);
        }
    } else
        args(wide ? realspace_cell_kernel<false, COUNT, true, true, FLD>
                  : realspace_cell_kernel<false, COUNT, true, false, FLD>);
    SE_LAUNCH_CHECK();
    pl->launches += 1;
    if (!full && !COUNT) {
        if (FLD)
            realspace_finish_field_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(
                acc, pl->cbin.idx_sorted.as<int>(), N, phi);
        else
            realspace_finish_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(acc, pl->cbin.rec.as<double4>(),
                                                                               pl->cbin.idx_sorted.as<int>(), N, a,
                                                                               phi);
        SE_LAUNCH_CHECK();
        pl->launches += 1;
    }
    if (!COUNT) prof_end(pl, SE_K_REALSPACE);
}

template <bool FLD>
static void realspace_impl(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi, int add_self,
                           int rank, int world) {
    const double L = pl->L, rc = pl->p.rc, xi = pl->p.xi;
    const int D = pl->D;
    const int nc = FLD ? 3 : 1;
    if (!(xi > 0) || !(rc > 0)) fail(SE_EINVAL, "xi and rc must be positive");
    cudaStream_t st = pl->stream;
    pl->flag.ensure(sizeof(int) * 4);
    SE_CUDA(cudaMemsetAsync(pl->flag.ptr, 0, sizeof(int) * 4, st));
    if (world > 1) SE_CUDA(cudaMemsetAsync(phi, 0, sizeof(double) * nc * (N > 0 ? N : 1), st));
    if (N <= 0) return;
    RealArgs a{};
    a.L = L;
    a.xi = xi;
    a.rc = rc;
    a.rc2 = rc * rc * (1.0 + 1e-12);  // prefilter only; the exact test is r < rc
    a.dense_min = dense_threshold();
    a.n_own = pl->dom.ncols > 0 ? pl->dom.n_own : -1;
    a.add_self = add_self;
    a.sqrtpi = std::sqrt(M_PI);
    a.rlo = N * rank / world;
    a.rhi = N * (rank + 1) / world;
    set_prefilter(a);
    fit_pair_poly(pl, a, FLD ? 1 : 0);
    if (D >= 1 && rc > L / 2 + 1e-12) {
        int layers = (int)std::floor((rc + L / 2) / L) + 1;
        prof_begin(pl, SE_K_REALSPACE);
        realspace_image_kernel<FLD><<<(unsigned)((N + 127) / 128), 128, 0, st>>>(pos, q, N, a.rlo, a.rhi, a, D, layers,
                                                                                phi, pl->flag.as<int>());
        SE_LAUNCH_CHECK();
        prof_end(pl, SE_K_REALSPACE);
        pl->launches += 1;
    } else {
        cell_bin(pl, pos, q, N, a, full_shell<FLD>(pl, a));
        launch_cell<false, FLD>(pl, N, a, phi, nullptr);
    }
}

void realspace_run(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi, int add_self, int rank,
                   int world) {
    realspace_impl<false>(pl, pos, q, N, phi, add_self, rank, world);
}

// Domain-decomposed real space: the local set = own particles (caller order
// [0, n_own), all in the columns cx in [col_lo, col_hi) of the ncols x ncols
// column grid) + halo particles (the columns up to `reach` beyond col_hi,
// +x side, periodic wrap on a periodic x).  Every unordered pair with one
// end in the own columns is evaluated once here or on the rank owning the
// other end (the half shell points to +x): phi[own] = the pair sums of the
// own particles (+ self term), phi[halo] = the Newton source-side sums of
// the halo particles, to be returned to their owners and added there.
void realspace_domain_run(se_plan *pl, const double *pos, const double *q, int64_t n_local, int64_t n_own, int ncols,
                          int col_lo, int col_hi, double *phi, int add_self) {
    if (pl->D >= 1 && pl->p.rc > pl->L / 2 + 1e-12) fail(SE_EINVAL, "domain mode covers the cell path (rc <= L/2)");
    if (ncols < 1 || col_lo < 0 || col_hi > ncols || col_lo > col_hi || n_own < 0 || n_own > n_local)
        fail(SE_EINVAL, "invalid domain (ncols, col_lo, col_hi, n_own)");
    pl->dom = DomainSpec{ncols, col_lo, col_hi, n_own};
    try {
        realspace_impl<false>(pl, pos, q, n_local, phi, add_self, 0, 1);
    } catch (...) {
        pl->dom = DomainSpec{};
        throw;
    }
    pl->dom = DomainSpec{};
}

// Real-space part of the electric field E_R = -grad phi_R at every particle
// (N x 3, caller order): sum over in-cutoff pairs of
// q_s (erfc(xi r)/r + (2 xi/sqrt(pi)) exp(-xi^2 r^2)) (x_t - x_s) / r^2,
// the same pair set, cell path and Newton symmetry as realspace_run.
void realspace_field_run(se_plan *pl, const double *pos, const double *q, int64_t N, double *E, int rank,
                         int world) {
    realspace_impl<true>(pl, pos, q, N, E, 0, rank, world);
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
    a.dense_min = kT * 32 + 1;  // counting: the compaction path counts exactly
    a.n_own = -1;
    a.sqrtpi = std::sqrt(M_PI);
    a.rlo = 0;
    a.rhi = N;
    set_prefilter(a);
    pl->flag.ensure(sizeof(int) * 4);
    SE_CUDA(cudaMemsetAsync(pl->flag.ptr, 0, sizeof(int) * 4, pl->stream));
    pl->pairs.ensure(sizeof(unsigned long long));
    SE_CUDA(cudaMemsetAsync(pl->pairs.ptr, 0, sizeof(unsigned long long), pl->stream));
    cell_bin(pl, pos, q, N, a, full_shell<false>(pl, a));
    launch_cell<true>(pl, N, a, nullptr, pl->pairs.as<unsigned long long>());
    unsigned long long h = 0;
    SE_CUDA(cudaMemcpyAsync(&h, pl->pairs.ptr, sizeof(h), cudaMemcpyDeviceToHost, pl->stream));
    SE_CUDA(cudaStreamSynchronize(pl->stream));
    *pairs = (long long)h;
}

}  // namespace se
