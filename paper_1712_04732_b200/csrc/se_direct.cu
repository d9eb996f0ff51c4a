// Direct Ewald sums on the device: the reference's independently coded
// evaluators (oracle.py) for large-N validation of the SE path (SURVEY.md
// 8(f).3).  Not on the hot path.
//
//  * D = 3, oracle.py:109-118: phi_m = (4 pi / L^3) sum_{k != 0}
//    e^{-k^2/4xi^2}/k^2 Re(e^{i k.x_m} S_k), S_k = sum_n q_n e^{-i k.x_n}, over
//    the integer modes |n_a| <= kmax.  S(-k) = conj S(k), so only the half
//    space (n1 > 0, or n1 = 0 and n2 > 0, or n1 = n2 = 0 and n3 > 0) is
//    formed, with weight 2.
//      structure_factor_kernel: one CTA per (n1, 16 rows of n2, 128 columns
//      of n3); particles staged 16 at a time as q e^{-i(k1 x + k2 y)} per row
//      and e^{-i k3 z} per column (sincospi of the reduced phase), each
//      thread accumulating 2 x 4 modes;
//      weight_kernel: W_k = 2 e^{-k^2/4xi^2}/k^2 S_k on the half space, 0
//      elsewhere;
//      potential_kernel: one target per thread, modes in storage order with
//      the n3 phase advanced by a rotation (rows restarted by sincospi).
//  * D = 0, oracle.py:181-192: phi_m = sum_{n != m} q_n erf(xi r)/r +
//    q_m 2 xi / sqrt(pi); coincident distinct particles are an error.
//  * D = 2, oracle.py:120-153: per periodic mode k = (n1, n2) 2 pi / L != 0 the
//    closed form (pi / L^2) sum_n q_n e^{i k.(x_m - x_n)} [e^{kz} erfc(k/2xi +
//    xi z) + e^{-kz} erfc(k/2xi - xi z)] / k, z = z_m - z_n, in its overflow-safe
//    erfcx form, minus (2 sqrt(pi) / L^2) sum_n q_n [e^{-xi^2 z^2}/xi +
//    sqrt(pi) z erf(xi z)]; one CTA per target, threads over sources, modes
//    over the half plane (weight 2) with e^{-k^2/4xi^2}, 1/k tabulated.
//  * D = 1, oracle.py:156-178: (1/L) sum_n q_n 2 sum_{j=1..kmax} cos(k_j x)
//    K0(a_j, b) - (1/L) sum_{n != m} q_n [gamma + ln b + E1(b)], x = x_m - x_n,
//    b = xi^2 |transverse distance|^2, a_j = k_j^2/4xi^2, with the incomplete
//    Bessel K0(a, b) = int_0^inf exp(-a e^u - b e^-u) du (oracle.py:41-55) by
//    Gauss-Legendre panels in u; the mode sum is moved under the integral
//    (e^{-a_j e^u} = q^{j^2}, q = e^{-a_1 e^u}: a recurrence per node).
#include <cstring>
#include <vector>

#include "se_common.h"

using namespace se;

#define SE_API_BEGIN try {
#define SE_API_END                            \
    return SE_OK;                             \
    }                                         \
    catch (const se::Error &e) {              \
        se::set_last_error(e.what());         \
        return e.code;                        \
    }                                         \
    catch (const std::exception &e) {         \
        se::set_last_error(e.what());         \
        return SE_EDEVICE;                    \
    }

namespace {

constexpr int kRows = 16, kCols = 128, kChunk = 16;  // 36 KB of static shared memory

// S[n1][n2 + kmax][n3 + kmax], n1 in [0, kmax]; row pitch P = 2 kmax + 1
__global__ void __launch_bounds__(256) structure_factor_kernel(const double *__restrict__ pos,
                                                               const double *__restrict__ q, int64_t N, double invL,
                                                               int kmax, double2 *__restrict__ S) {
    __shared__ double2 qab[kChunk][kRows];
    __shared__ double2 cz[kChunk][kCols];
    const int P = 2 * kmax + 1;
    const int n1 = blockIdx.x;
    const int r0 = blockIdx.y * kRows, c0 = blockIdx.z * kCols;
    const int tid = threadIdx.x, ty = tid >> 5, tx = tid & 31;
    double2 acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
    for (int64_t p0 = 0; p0 < N; p0 += kChunk) {
        const int np = (int)min((int64_t)kChunk, N - p0);
        __syncthreads();
        // rows: q e^{-2 pi i (n1 x + n2 y)/L}; columns: e^{-2 pi i n3 z / L}
        for (int e = tid; e < kChunk * (kRows + kCols); e += 256) {
            const int p = e / (kRows + kCols), j = e % (kRows + kCols);
            double2 v = make_double2(0.0, 0.0);
            if (p < np) {
                const int64_t n = p0 + p;
                double s, c;
                if (j < kRows) {
                    const int n2 = r0 + j - kmax;
                    const double ph = -2.0 * ((double)n1 * pos[3 * n] + (double)n2 * pos[3 * n + 1]) * invL;
                    sincospi(ph, &s, &c);
                    const double qn = q[n];
                    v = make_double2(qn * c, qn * s);
                } else {
                    const int n3 = c0 + (j - kRows) - kmax;
                    sincospi(-2.0 * (double)n3 * pos[3 * n + 2] * invL, &s, &c);
                    v = make_double2(c, s);
                }
            }
            if (j < kRows)
                qab[p][j] = v;
            else
                cz[p][j - kRows] = v;
        }
        __syncthreads();
        for (int p = 0; p < np; ++p) {
            const double2 a0 = qab[p][2 * ty], a1 = qab[p][2 * ty + 1];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double2 c = cz[p][tx + 32 * b];
                acc[0][b].x = fma(a0.x, c.x, fma(-a0.y, c.y, acc[0][b].x));
                acc[0][b].y = fma(a0.x, c.y, fma(a0.y, c.x, acc[0][b].y));
                acc[1][b].x = fma(a1.x, c.x, fma(-a1.y, c.y, acc[1][b].x));
                acc[1][b].y = fma(a1.x, c.y, fma(a1.y, c.x, acc[1][b].y));
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        const int row = r0 + 2 * ty + a;
        if (row >= P) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int col = c0 + tx + 32 * b;
            if (col < P) S[((int64_t)n1 * P + row) * P + col] = acc[a][b];
        }
    }
}

__global__ void weight_kernel(double2 *__restrict__ S, int kmax, double twopi_L, double inv4xi2) {
    const int P = 2 * kmax + 1;
    const int64_t total = (int64_t)(kmax + 1) * P * P;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int n3 = (int)(i % P) - kmax, n2 = (int)((i / P) % P) - kmax, n1 = (int)(i / ((int64_t)P * P));
        const bool half = n1 > 0 || (n1 == 0 && (n2 > 0 || (n2 == 0 && n3 > 0)));
        double w = 0.0;
        if (half) {
            const double k2 = twopi_L * twopi_L * ((double)n1 * n1 + (double)n2 * n2 + (double)n3 * n3);
            w = 2.0 * exp(-k2 * inv4xi2) / k2;
        }
        S[i] = make_double2(S[i].x * w, S[i].y * w);
    }
}

__global__ void __launch_bounds__(256) potential_kernel(const double *__restrict__ pos,
                                                        const int64_t *__restrict__ targets, int64_t T, double invL,
                                                        int kmax, const double2 *__restrict__ W, double scale,
                                                        double *__restrict__ phi) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    const int64_t m = targets ? targets[t] : t;
    const double x = pos[3 * m], y = pos[3 * m + 1], z = pos[3 * m + 2];
    const int P = 2 * kmax + 1;
    double sz, cz, s0, c0;
    sincospi(2.0 * z * invL, &sz, &cz);                 // e^{+i 2 pi z / L}: step along n3
    sincospi(-2.0 * (double)kmax * z * invL, &s0, &c0);  // n3 = -kmax
    double acc = 0.0;
    const double2 *w = W;
    for (int n1 = 0; n1 <= kmax; ++n1) {
        for (int n2 = -kmax; n2 <= kmax; ++n2) {
            double sa, ca;
            sincospi(2.0 * ((double)n1 * x + (double)n2 * y) * invL, &sa, &ca);
            // e = e^{i(k1 x + k2 y)} e^{i k3 z}, advanced by the n3 step
            double er = ca * c0 - sa * s0, ei = ca * s0 + sa * c0;
            for (int c = 0; c < P; ++c) {
                const double2 v = w[c];
                acc = fma(er, v.x, fma(-ei, v.y, acc));
                const double nr = er * cz - ei * sz;
                ei = er * sz + ei * cz;
                er = nr;
            }
            w += P;
        }
    }
    phi[t] = scale * acc;
}

__global__ void __launch_bounds__(256) erf_pair_kernel(const double *__restrict__ pos, const double *__restrict__ q,
                                                       int64_t N, const int64_t *__restrict__ targets, int64_t T,
                                                       double xi, double *__restrict__ phi, int *__restrict__ flag) {
    __shared__ double4 src[256];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = t < T;
    const int64_t m = live ? (targets ? targets[t] : t) : -1;
    const double x = live ? pos[3 * m] : 0.0, y = live ? pos[3 * m + 1] : 0.0, z = live ? pos[3 * m + 2] : 0.0;
    double acc = 0.0;
    int bad = 0;
    for (int64_t j0 = 0; j0 < N; j0 += 256) {
        __syncthreads();
        const int64_t j = j0 + threadIdx.x;
        if (j < N) src[threadIdx.x] = make_double4(pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], q[j]);
        __syncthreads();
        const int nj = (int)min((int64_t)256, N - j0);
        if (!live) continue;
        for (int k = 0; k < nj; ++k) {
            const double4 s = src[k];
            const double dx = x - s.x, dy = y - s.y, dz = z - s.z;
            const double r = sqrt(fma(dz, dz, fma(dy, dy, dx * dx)));
            if (j0 + k == m) continue;
            if (r < 1e-14) {
                bad = 1;
                continue;
            }
            acc += s.w * erf(xi * r) / r;
        }
    }
    if (bad) atomicExch(flag, 1);
    if (live) phi[t] = acc + q[m] * (2.0 * xi / sqrt(M_PI));
}

struct Mode2 {
    double k, ek, invk;  // |k|, e^{-k^2/4xi^2}, 1/|k|
    int n1, n2;
};

__global__ void __launch_bounds__(256) direct2p_kernel(const double *__restrict__ pos, const double *__restrict__ q,
                                                       int64_t N, const int64_t *__restrict__ targets, double L,
                                                       double xi, const Mode2 *__restrict__ modes, int nmodes,
                                                       double *__restrict__ phi) {
    const int64_t m = targets ? targets[blockIdx.x] : (int64_t)blockIdx.x;
    const double xm = pos[3 * m], ym = pos[3 * m + 1], zm = pos[3 * m + 2];
    const double twopiL = 2.0 * M_PI / L, inv2xi = 0.5 / xi;
    double acc = 0.0, zero = 0.0;
    for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
        const double dx = xm - pos[3 * n], dy = ym - pos[3 * n + 1], z = zm - pos[3 * n + 2];
        const double qn = q[n];
        const double ez = exp(-(xi * z) * (xi * z));
        zero += qn * (ez / xi + sqrt(M_PI) * z * erf(xi * z));
        double s = 0.0;
        for (int j = 0; j < nmodes; ++j) {
            const Mode2 md = modes[j];
            const double u1 = md.k * inv2xi + xi * z, u2 = md.k * inv2xi - xi * z;
            const double g = md.ek * ez;  // e^{guard}, guard = -(k^2/4xi^2 + xi^2 z^2)
            const double b1 = u1 >= 0.0 ? erfcx(u1) * g : exp(md.k * z) * erfc(u1);
            const double b2 = u2 >= 0.0 ? erfcx(u2) * g : exp(-md.k * z) * erfc(u2);
            const double ph = twopiL * (md.n1 * dx + md.n2 * dy);
            s += cos(ph) * (b1 + b2) * md.invk;
        }
        acc += qn * s;
    }
    __shared__ double ra[256], rz[256];
    ra[threadIdx.x] = acc;
    rz[threadIdx.x] = zero;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            ra[threadIdx.x] += ra[threadIdx.x + o];
            rz[threadIdx.x] += rz[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        phi[blockIdx.x] = (M_PI / (L * L)) * 2.0 * ra[0] - (2.0 * sqrt(M_PI) / (L * L)) * rz[0];
}

// E1(x), x > 0: power series for x <= 1, modified Lentz continued fraction
// above (oracle.py:58-91 uses the same two regimes).
__device__ double e1_dev(double x) {
    if (x <= 1.0) {
        double total = -0.5772156649015328606 - log(x), term = 1.0;
        for (int k = 1; k < 60; ++k) {
            term *= -x / k;
            const double c = -term / k;
            total += c;
            if (fabs(c) < 1e-18 * fabs(total)) break;
        }
        return total;
    }
    const double tiny = 1e-300;
    double b = x + 1.0, c = 1.0 / tiny, d = 1.0 / b, f = d;
    for (int k = 1; k < 300; ++k) {
        const double an = -(double)k * k;
        b += 2.0;
        d = 1.0 / (b + an * d);
        c = b + an / c;
        const double delta = c * d;
        f *= delta;
        if (fabs(delta - 1.0) < 1e-16) break;
    }
    return exp(-x) * f;
}

struct Node1 {
    double emu, w, q;  // e^{-u}, weight, e^{-a_1 e^u}
};

__global__ void __launch_bounds__(256) direct1p_kernel(const double *__restrict__ pos, const double *__restrict__ q,
                                                       int64_t N, const int64_t *__restrict__ targets, double L,
                                                       double xi, int kmax, const Node1 *__restrict__ nodes,
                                                       int nnodes, double *__restrict__ phi, int *__restrict__ flag) {
    const int64_t m = targets ? targets[blockIdx.x] : (int64_t)blockIdx.x;
    const double xm = pos[3 * m], ym = pos[3 * m + 1], zm = pos[3 * m + 2];
    double acc = 0.0, zero = 0.0;
    int bad = 0;
    for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
        const double x = xm - pos[3 * n], dy = ym - pos[3 * n + 1], dz = zm - pos[3 * n + 2];
        const double w2 = dy * dy + dz * dz;
        if (n != m && w2 < 1e-28) {
            bad = 1;
            continue;
        }
        const double b = xi * xi * w2, qn = q[n];
        const double c1 = cos(2.0 * M_PI * x / L);
        double s = 0.0;
        for (int j = 0; j < nnodes; ++j) {
            const Node1 nd = nodes[j];
            const double eb = exp(-b * nd.emu);
            if (eb == 0.0) continue;
            // sum_i cos(i theta) q^{i^2}, i = 1..kmax
            const double qq = nd.q * nd.q;
            double t = nd.q, p = nd.q * qq;  // q^{i^2}, q^{2i+1}
            double cm = 1.0, ci = c1, sum = 0.0;
            for (int i = 1; i <= kmax && t > 1e-30; ++i) {
                sum = fma(ci, t, sum);
                t *= p;
                p *= qq;
                const double cn = 2.0 * c1 * ci - cm;
                cm = ci;
                ci = cn;
            }
            s = fma(nd.w * eb, sum, s);
        }
        acc = fma(qn, 2.0 * s, acc);
        if (n != m) zero += qn * (0.5772156649015328606 + log(b) + e1_dev(b));
    }
    __shared__ double ra[256], rz[256];
    ra[threadIdx.x] = acc;
    rz[threadIdx.x] = zero;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            ra[threadIdx.x] += ra[threadIdx.x + o];
            rz[threadIdx.x] += rz[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (bad) atomicExch(flag, 1);
    if (threadIdx.x == 0) phi[blockIdx.x] = (ra[0] - rz[0]) / L;
}

void check_common(int64_t N, int64_t T, const double *pos) {
    if (N < 0 || T < 0) fail(SE_EINVAL, "negative particle or target count");
    if (N > 0 && !pos) fail(SE_EINVAL, "null positions");
}

struct DevBuf {
    void *p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes) SE_CUDA(cudaMalloc(&p, bytes));
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

void require_device() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        fail(SE_EDEVICE, "no CUDA device available (the SE B200 library has no CPU fallback)");
    }
}

void direct_3p(const double *pos, const double *q, int64_t N, double L, double xi, int kmax,
               const int64_t *targets, int64_t T, double *phi, cudaStream_t st) {
    check_common(N, T, pos);
    if (!(L > 0) || !(xi > 0)) fail(SE_EINVAL, "L and xi must be positive");
    if (kmax < 1 || kmax > 1000) fail(SE_EINVAL, "kmax must lie in [1, 1000]");
    if (T == 0) return;
    const int P = 2 * kmax + 1;
    DevBuf S(sizeof(double2) * (size_t)(kmax + 1) * P * P);
    const double invL = 1.0 / L;
    dim3 grid((unsigned)(kmax + 1), (unsigned)((P + kRows - 1) / kRows), (unsigned)((P + kCols - 1) / kCols));
    structure_factor_kernel<<<grid, 256, 0, st>>>(pos, q, N, invL, kmax, (double2 *)S.p);
    SE_LAUNCH_CHECK();
    weight_kernel<<<1184, 256, 0, st>>>((double2 *)S.p, kmax, 2.0 * M_PI / L, 1.0 / (4.0 * xi * xi));
    SE_LAUNCH_CHECK();
    potential_kernel<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(pos, targets, T, invL, kmax,
                                                                 (const double2 *)S.p, 4.0 * M_PI / (L * L * L), phi);
    SE_LAUNCH_CHECK();
    SE_CUDA(cudaStreamSynchronize(st));
}

void direct_0p(const double *pos, const double *q, int64_t N, double xi, const int64_t *targets, int64_t T,
               double *phi, cudaStream_t st) {
    check_common(N, T, pos);
    if (!(xi > 0)) fail(SE_EINVAL, "xi must be positive");
    if (T == 0) return;
    DevBuf flag(sizeof(int));
    SE_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    erf_pair_kernel<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(pos, q, N, targets, T, xi, phi, (int *)flag.p);
    SE_LAUNCH_CHECK();
    int h = 0;
    SE_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SE_CUDA(cudaStreamSynchronize(st));
    if (h) fail(SE_ESINGULAR, "coincident distinct particles");
}

void direct_2p(const double *pos, const double *q, int64_t N, double L, double xi, int kmax,
               const int64_t *targets, int64_t T, double *phi, cudaStream_t st) {
    check_common(N, T, pos);
    if (!(L > 0) || !(xi > 0)) fail(SE_EINVAL, "L and xi must be positive");
    if (kmax < 1 || kmax > 1000) fail(SE_EINVAL, "kmax must lie in [1, 1000]");
    if (T == 0) return;
    std::vector<Mode2> md;
    for (int n1 = 0; n1 <= kmax; ++n1)
        for (int n2 = -kmax; n2 <= kmax; ++n2) {
            if (n1 == 0 && n2 <= 0) continue;  // half plane, weight 2
            const double k = 2.0 * M_PI / L * std::sqrt((double)n1 * n1 + (double)n2 * n2);
            md.push_back(Mode2{k, std::exp(-k * k / (4.0 * xi * xi)), 1.0 / k, n1, n2});
        }
    DevBuf dm(sizeof(Mode2) * md.size());
    SE_CUDA(cudaMemcpyAsync(dm.p, md.data(), sizeof(Mode2) * md.size(), cudaMemcpyHostToDevice, st));
    direct2p_kernel<<<(unsigned)T, 256, 0, st>>>(pos, q, N, targets, L, xi, (const Mode2 *)dm.p, (int)md.size(),
                                                 phi);
    SE_LAUNCH_CHECK();
    SE_CUDA(cudaStreamSynchronize(st));
}

// Gauss-Legendre nodes on [-1, 1] (Newton on the Legendre recurrence, host)
static void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
    x.resize(n);
    w.resize(n);
    for (int i = 0; i < n; ++i) {
        double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;
            for (int j = 2; j <= n; ++j) {
                const double p2 = ((2 * j - 1) * z * p1 - (j - 1) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (z * p1 - p0) / (z * z - 1.0);
            const double dz = p1 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-16) break;
        }
        x[i] = z;
        w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
}

void direct_1p(const double *pos, const double *q, int64_t N, double L, double xi, int kmax,
               const int64_t *targets, int64_t T, double *phi, cudaStream_t st) {
    check_common(N, T, pos);
    if (!(L > 0) || !(xi > 0)) fail(SE_EINVAL, "L and xi must be positive");
    if (kmax < 1 || kmax > 1000) fail(SE_EINVAL, "kmax must lie in [1, 1000]");
    if (T == 0) return;
    // u in [0, U]: e^{-a_1 e^U} < e^{-46}; panels of width 1/2, 20 points each
    const double k1 = 2.0 * M_PI / L, a1 = k1 * k1 / (4.0 * xi * xi);
    const double U = std::log(46.0 / a1) > 0.5 ? std::log(46.0 / a1) : 0.5;
    const int npan = (int)std::ceil(U / 0.5);
    std::vector<double> gx, gw;
    gauss_legendre(20, gx, gw);
    std::vector<Node1> nodes;
    for (int pnl = 0; pnl < npan; ++pnl) {
        const double lo = U * pnl / npan, hi = U * (pnl + 1) / npan;
        for (int i = 0; i < 20; ++i) {
            const double u = 0.5 * (lo + hi) + 0.5 * (hi - lo) * gx[i];
            nodes.push_back(Node1{std::exp(-u), 0.5 * (hi - lo) * gw[i], std::exp(-a1 * std::exp(u))});
        }
    }
    DevBuf dn(sizeof(Node1) * nodes.size()), flag(sizeof(int));
    SE_CUDA(cudaMemcpyAsync(dn.p, nodes.data(), sizeof(Node1) * nodes.size(), cudaMemcpyHostToDevice, st));
    SE_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    direct1p_kernel<<<(unsigned)T, 256, 0, st>>>(pos, q, N, targets, L, xi, kmax, (const Node1 *)dn.p,
                                                 (int)nodes.size(), phi, (int *)flag.p);
    SE_LAUNCH_CHECK();
    int h = 0;
    SE_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SE_CUDA(cudaStreamSynchronize(st));
    if (h) fail(SE_ESINGULAR, "two charges share transverse coordinates; the zero-mode log diverges");
}

// host buffers -> device, run, phi back
template <class F>
void via_device(const double *pos, const double *q, int64_t N, const int64_t *targets, int64_t T, double *phi,
                F &&run) {
    require_device();
    const int64_t nt = targets ? T : N;
    DevBuf dpos(sizeof(double) * 3 * (size_t)N), dq(sizeof(double) * (size_t)N),
        dt(targets ? sizeof(int64_t) * (size_t)T : 0), dphi(sizeof(double) * (size_t)nt);
    if (N) {
        SE_CUDA(cudaMemcpy(dpos.p, pos, sizeof(double) * 3 * N, cudaMemcpyHostToDevice));
        SE_CUDA(cudaMemcpy(dq.p, q, sizeof(double) * N, cudaMemcpyHostToDevice));
    }
    if (targets && T) SE_CUDA(cudaMemcpy(dt.p, targets, sizeof(int64_t) * T, cudaMemcpyHostToDevice));
    run((const double *)dpos.p, (const double *)dq.p, (const int64_t *)dt.p, nt, (double *)dphi.p);
    if (nt) SE_CUDA(cudaMemcpy(phi, dphi.p, sizeof(double) * nt, cudaMemcpyDeviceToHost));
}

void check_targets_host(const int64_t *targets, int64_t T, int64_t N) {
    if (!targets) return;
    for (int64_t i = 0; i < T; ++i)
        if (targets[i] < 0 || targets[i] >= N) fail(SE_EINVAL, "target index out of range");
}

}  // namespace

extern "C" {

int se_direct_kspace_3p_dev(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                            const int64_t *targets, int64_t T, double *phi, void *stream) {
    SE_API_BEGIN
    direct_3p(pos, q, N, L, xi, kmax, targets, targets ? T : N, phi, (cudaStream_t)stream);
    SE_API_END
}

int se_direct_kspace_3p_host(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                             const int64_t *targets, int64_t T, double *phi) {
    SE_API_BEGIN
    check_targets_host(targets, T, N);
    via_device(pos, q, N, targets, T, phi,
               [&](const double *dp, const double *dq, const int64_t *dt, int64_t nt, double *dphi) {
                   direct_3p(dp, dq, N, L, xi, kmax, targets ? dt : nullptr, nt, dphi, 0);
               });
    SE_API_END
}

int se_direct_kspace_0p_dev(const double *pos, const double *q, int64_t N, double xi, const int64_t *targets,
                            int64_t T, double *phi, void *stream) {
    SE_API_BEGIN
    direct_0p(pos, q, N, xi, targets, targets ? T : N, phi, (cudaStream_t)stream);
    SE_API_END
}

int se_direct_kspace_0p_host(const double *pos, const double *q, int64_t N, double xi, const int64_t *targets,
                             int64_t T, double *phi) {
    SE_API_BEGIN
    check_targets_host(targets, T, N);
    via_device(pos, q, N, targets, T, phi,
               [&](const double *dp, const double *dq, const int64_t *dt, int64_t nt, double *dphi) {
                   direct_0p(dp, dq, N, xi, targets ? dt : nullptr, nt, dphi, 0);
               });
    SE_API_END
}

int se_direct_kspace_2p_dev(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                            const int64_t *targets, int64_t T, double *phi, void *stream) {
    SE_API_BEGIN
    direct_2p(pos, q, N, L, xi, kmax, targets, targets ? T : N, phi, (cudaStream_t)stream);
    SE_API_END
}

int se_direct_kspace_2p_host(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                             const int64_t *targets, int64_t T, double *phi) {
    SE_API_BEGIN
    check_targets_host(targets, T, N);
    via_device(pos, q, N, targets, T, phi,
               [&](const double *dp, const double *dq, const int64_t *dt, int64_t nt, double *dphi) {
                   direct_2p(dp, dq, N, L, xi, kmax, targets ? dt : nullptr, nt, dphi, 0);
               });
    SE_API_END
}

int se_direct_kspace_1p_dev(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                            const int64_t *targets, int64_t T, double *phi, void *stream) {
    SE_API_BEGIN
    direct_1p(pos, q, N, L, xi, kmax, targets, targets ? T : N, phi, (cudaStream_t)stream);
    SE_API_END
}

int se_direct_kspace_1p_host(const double *pos, const double *q, int64_t N, double L, double xi, int32_t kmax,
                             const int64_t *targets, int64_t T, double *phi) {
    SE_API_BEGIN
    check_targets_host(targets, T, N);
    via_device(pos, q, N, targets, T, phi,
               [&](const double *dp, const double *dq, const int64_t *dt, int64_t nt, double *dphi) {
                   direct_1p(dp, dq, N, L, xi, kmax, targets ? dt : nullptr, nt, dphi, 0);
               });
    SE_API_END
}

}  // extern "C"
