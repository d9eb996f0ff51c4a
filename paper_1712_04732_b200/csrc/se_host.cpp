// Host-side planning for the SE B200 library: parameter validation, grid
// geometry, FFT padding sizes, mode partitions, and the small 1-D tables
// (window transforms, truncated Green's functions) that the device kernels
// consume.  These are plan-time computations (microseconds), the analogue of
// the reference's Grid.build / padded_size / windows.fourier /
// greens.zero_mode_values; no per-particle or per-grid-point work runs here.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "se_common.h"

namespace se {

static thread_local std::string g_last_error;
void set_last_error(const std::string &msg) { g_last_error = msg; }

// ------------------------------------------------------------- FFT sizes
static bool smooth7(int m) {
    for (int p : {2, 3, 5, 7})
        while (m % p == 0) m /= p;
    return m == 1;
}

// aft.py:68-73
int next_even_smooth(int n) {
    int m = n < 2 ? 2 : n;
    while ((m & 1) || !smooth7(m)) ++m;
    return m;
}

// aft.py:76-84
int padded_size(double s, int n) {
    if (s < 1.0) fail(SE_EINVAL, "upsampling factor must be >= 1");
    double t = std::ceil(s * n - 1e-9);
    int want = (int)t;
    if (want <= n) return n;
    return next_even_smooth(want);
}

// core.py:118-138
void validate(const se_params_t &p, double L, int D) {
    if (D < 0 || D > 3) fail(SE_EINVAL, "D must be in {0,1,2,3}, got " + std::to_string(D));
    if (!(L > 0)) fail(SE_EINVAL, "box length must be positive");
    if (!(p.xi > 0)) fail(SE_EINVAL, "xi must be positive");
    if (!(p.rc > 0)) fail(SE_EINVAL, "rc must be positive");
    if (p.M < 2 || p.M % 2) fail(SE_EINVAL, "M must be an even integer >= 2");
    if (!(1 <= p.P && p.P <= p.M)) fail(SE_EINVAL, "P must satisfy 1 <= P <= M");
    if (p.window < 0 || p.window > 2) fail(SE_EINVAL, "unknown window");
    if (!(p.shape > 0)) fail(SE_EINVAL, "shape parameter must be positive");
    if (p.s0 < 1.0 || p.s < 1.0) fail(SE_EINVAL, "upsampling factors must be >= 1");
    if (!(0 <= p.nI && p.nI <= p.M / 2)) fail(SE_EINVAL, "nI must lie in [0, M/2]");
    if ((D == 1 || D == 2) && (p.M + p.P) % 2) fail(SE_EINVAL, "M + P must be even when 0 < D < 3");
    if (D < 3 && !(p.R > 0)) fail(SE_EINVAL, "R must be positive for D < 3");
}

// sekspace.py:53-70
se_grid_t build_grid(int D, double L, const se_params_t &p) {
    se_grid_t g{};
    g.D = D;
    g.M = p.M;
    g.P = p.P;
    g.L = L;
    g.h = L / p.M;
    g.Mt = p.M + p.P;
    g.Lt = L + p.P * g.h;
    g.R = D < 3 ? p.R : 0.0;
    g.g0 = D < 3 ? padded_size(p.s0, g.Mt) : p.M;
    g.gs = (D == 1 || D == 2) ? padded_size(p.s, g.Mt) : g.Mt;
    for (int a = 0; a < 3; ++a) {
        g.shape[a] = a < D ? p.M : g.Mt;
        g.offsets[a] = a < D ? 0.0 : 0.5 * p.P * g.h;
    }
    return g;
}

// sekspace.py:266-279 (precompute_truncated_greens geometry)
D0Geom d0_geometry(double L, int M, int P, double s0, double rc, bool has_rc) {
    if (s0 < 1.0 + std::sqrt(3.0) - 1e-12)
        fail(SE_EINVAL, "free-space precompute requires s0 >= 1 + sqrt(3)");
    double h = L / M;
    int Mt = M + P;
    double Lt = L + P * h;
    double reach = has_rc ? std::fmin(rc, L) : 0.0;
    double margin = std::fmax(P * h, reach);
    int nhalf = (int)std::ceil((L + margin) / h - 0.5);
    int a = 2 * nhalf, b = 2 * Mt;
    D0Geom out;
    out.nconv = next_even_smooth(a > b ? a : b);
    double W = (out.nconv / 2) * h;
    out.R = std::sqrt(3.0) * L + margin;
    double s0b = std::fmax(s0, (W + out.R) / Lt);
    out.g0 = padded_size(s0b, Mt);
    return out;
}

// aft.py:56-58
std::vector<int> signed_modes(int n) {
    std::vector<int> m(n);
    for (int j = 0; j < n; ++j) m[j] = j < (n + 1) / 2 ? j : j - n;
    return m;
}

// sekspace.py:100-102: 2 pi fftfreq(n, d=h) -- numpy computes
// results = ints * (1/(n*d)) then multiplies by 2 pi.
std::vector<double> wavenumbers(int n, double h) {
    std::vector<int> m = signed_modes(n);
    std::vector<double> k(n);
    double val = 1.0 / (n * h);
    for (int j = 0; j < n; ++j) k[j] = 2.0 * M_PI * (m[j] * val);
    return k;
}

// ----------------------------------------------------------- special fns
// I0 by its power series in long double (all terms positive: no cancellation).
static long double bessel_i0_ld(long double x) {
    long double q = 0.25L * x * x, term = 1.0L, sum = 1.0L;
    for (int k = 1; k < 2000; ++k) {
        term *= q / ((long double)k * (long double)k);
        sum += term;
        if (term < sum * 1e-21L) break;
    }
    return sum;
}

double bessel_i0(double x) { return (double)bessel_i0_ld((long double)x); }

// windows.py:74-84, 106-112, 148-154
double window_value(int window, double w, double shape, double x) {
    if (!(std::fabs(x) <= w)) return 0.0;
    if (window == SE_WINDOW_GAUSSIAN) {
        double peak = shape / (w * std::sqrt(2.0 * M_PI));
        return peak * std::exp(-(shape * shape) * (x * x) / (2.0 * w * w));
    }
    double r = x / w;
    double t = 1.0 - r * r;
    if (t < 0.0) t = 0.0;
    if (window == SE_WINDOW_KB)
        return (double)(bessel_i0_ld((long double)(shape * std::sqrt(t))) / bessel_i0_ld((long double)shape));
    return std::exp(shape * (std::sqrt(t) - 1.0));
}

// Gauss-Legendre rule in extended precision (windows.py:184-199: nodes
// polished in np.longdouble).
static void gauss_legendre_ld(int n, std::vector<long double> &x, std::vector<long double> &wt) {
    x.resize(n);
    wt.resize(n);
    for (int i = 0; i < n; ++i) {
        long double z = std::cos(M_PIl * (i + 0.75L) / (n + 0.5L));
        long double dp = 0;
        for (int it = 0; it < 100; ++it) {
            long double p0 = 1.0L, p1 = z;
            for (int j = 2; j <= n; ++j) {
                long double p2 = ((2 * j - 1) * z * p1 - (j - 1) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (z * p1 - p0) / (z * z - 1.0L);
            long double dz = p1 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-21L) break;
        }
        long double p0 = 1.0L, p1 = z;
        for (int j = 2; j <= n; ++j) {
            long double p2 = ((2 * j - 1) * z * p1 - (j - 1) * p0) / j;
            p0 = p1;
            p1 = p2;
        }
        dp = n * (z * p1 - p0) / (z * z - 1.0L);
        x[n - 1 - i] = z;  // ascending order like leggauss
        wt[n - 1 - i] = 2.0L / ((1.0L - z * z) * dp * dp);
    }
}

// windows.py:202-211: 2w int_0^{pi/2} e^{beta(cos t - 1)} cos(k w sin t) cos t dt
static std::vector<double> bm_quadrature(double w, double beta, const std::vector<double> &k, int nodes) {
    std::vector<long double> x, wt;
    gauss_legendre_ld(nodes, x, wt);
    const long double q = (long double)(0.25 * M_PI);  // np.longdouble(0.25*math.pi)
    std::vector<long double> f(nodes), st(nodes);
    for (int i = 0; i < nodes; ++i) {
        long double th = q * (x[i] + 1.0L);
        long double c = std::cos(th);
        f[i] = std::exp((long double)beta * (c - 1.0L)) * c * (wt[i] * q);
        st[i] = std::sin(th);
    }
    std::vector<double> out(k.size());
    for (size_t j = 0; j < k.size(); ++j) {
        long double kw = (long double)k[j] * (long double)w;
        long double acc = 0.0L;
        for (int i = 0; i < nodes; ++i) acc += std::cos(kw * st[i]) * f[i];
        out[j] = (double)(2.0L * (long double)w * acc);
    }
    return out;
}

// windows.py:115-132: sinh(sqrt(rho2))/sqrt(rho2), continued to rho2 < 0 as
// sin(sqrt(-rho2))/sqrt(-rho2); a short Taylor series across the seam.
static double kb_sinhc(double rho2) {
    if (std::fabs(rho2) < 1e-6)
        return 1.0 + rho2 / 6.0 + rho2 * rho2 / 120.0 + rho2 * rho2 * rho2 / 5040.0;
    if (rho2 > 0) {
        double r = std::sqrt(rho2);
        return std::sinh(r) / r;
    }
    double r = std::sqrt(-rho2);
    return std::sin(r) / r;
}

// windows.py:87-91, 115-145, 214-239
std::vector<double> window_fourier(int window, int P, double h, double shape, const std::vector<double> &k) {
    double w = 0.5 * P * h;
    std::vector<double> out(k.size());
    if (window == SE_WINDOW_GAUSSIAN) {
        for (size_t j = 0; j < k.size(); ++j) {
            double a = w * k[j];
            out[j] = std::exp(-(a * a) / (2.0 * shape * shape));
        }
        return out;
    }
    if (window == SE_WINDOW_KB) {
        double i0b = (double)bessel_i0_ld((long double)shape);
        for (size_t j = 0; j < k.size(); ++j) {
            double kw = k[j] * w;
            out[j] = 2.0 * w * kb_sinhc(shape * shape - kw * kw) / i0b;
        }
        return out;
    }
    double kmax = 0.0;
    for (double v : k) kmax = std::fmax(kmax, std::fabs(v));
    int nodes = (int)(0.75 * (kmax * w + shape)) + 32;
    if (nodes < 64) nodes = 64;
    std::vector<double> vals = bm_quadrature(w, shape, k, nodes);
    std::vector<double> check = bm_quadrature(w, shape, k, 2 * nodes);
    double scale = 1e-300, dev = 0.0;
    for (size_t j = 0; j < k.size(); ++j) {
        scale = std::fmax(scale, std::fabs(check[j]));
        dev = std::fmax(dev, std::fabs(vals[j] - check[j]));
    }
    if (dev > 1e-13 * scale) fail(SE_ENUMERIC, "BM transform quadrature did not converge");
    return check;
}

// greens.py:48-85 (D=2 keeps the reference's sign, greens.py:75-82)
double greens_zero_mode(int D, double R, double kappa) {
    kappa = std::fabs(kappa);
    double t = R * kappa;
    if (t < 1e-2) {
        double z = t * t;
        if (D == 0)
            return R * R * (0.5 - z / 24.0 + z * z / 720.0 - z * z * z / 40320.0 + z * z * z * z / 3628800.0);
        if (D == 1) {
            double lr = std::log(R);
            return R * R * ((0.25 - 0.5 * lr) - z * (1.0 / 64.0 - lr / 16.0)
                            + z * z * (1.0 / 2304.0 - lr / 384.0)
                            - z * z * z * (1.0 / 147456.0 - lr / 18432.0)
                            + z * z * z * z * (1.0 / 14745600.0 - lr / 1474560.0));
        }
        return R * R * (-0.5 + z / 8.0 - z * z / 144.0 + z * z * z / 5760.0 - z * z * z * z / 403200.0);
    }
    if (D == 0) return R * R * (1.0 - std::cos(t)) / (t * t);
    if (D == 1) return (1.0 - ::j0(t)) / (kappa * kappa) - (R * std::log(R)) * ::j1(t) / kappa;
    return R * R * (1.0 - std::cos(t) - t * std::sin(t)) / (t * t);
}

// Polynomial pair term of the real-space kernel (se_realspace.cu, pair_poly):
// Q(t) = xi P(xi^2 rc^2 (t + 1)/2), P(s) = erf(sqrt s)/sqrt s, t in [-1, 1],
// as the Chebyshev interpolant (long double) of the smallest degree in
// {20, 24, 28, 32} whose interpolation error, checked on 513 points, stays
// below a quarter ulp of Q(0) = 2 xi / sqrt(pi) (the rounding of the
// coefficients to double then adds ~1 ulp of Q, |coefficients| < Q(0) --
// comparable to the rounding of 1/r at the cutoff).  Monomial coefficients
// in t go to pc[0..32]; returns the degree, 0 if none suffices (xi rc > ~5).
// kind 1: the field's R = Q - (2 xi/sqrt pi) exp(-xi^2 u) instead of Q.
static long double pair_P(long double s) {
    if (s <= 0.0L) return 2.0L / std::sqrt(3.14159265358979323846264338327950288L);
    const long double x = std::sqrt(s);
    return std::erf(x) / x;
}

int pair_poly_fit(double xi_, double rc_, int kind, double *pc) {
    static constexpr int kDegrees[] = {20, 24, 28, 32};
    const long double xi = xi_, S = (long double)xi_ * xi_ * rc_ * rc_;
    const long double pi = 3.14159265358979323846264338327950288L;
    // kind 1 (field): R = Q - (2 xi / sqrt pi) exp(-s), the factor of
    // g = (erfc(x)/r + (2 xi/sqrt pi) exp(-x^2))/r^2 = (1/r^2)(1/r - R)
    const long double c2 = 2.0L / std::sqrt(pi);
    auto fq = [&](long double t) {
        const long double s = S * (t + 1.0L) / 2.0L;
        return xi * (pair_P(s) - (kind == 1 ? c2 * std::exp(-s) : 0.0L));
    };
    const long double qtol = std::ldexp(1.0L, -54) * xi * c2;  // a quarter ulp of Q(0) = 2 xi / sqrt(pi)
    // SE_B200_PAIR_TOL_SCALE (A/B measurements only): a looser fit target
    static const long double tscale = [] {
        const char *e = std::getenv("SE_B200_PAIR_TOL_SCALE");
        return e ? (long double)std::atof(e) : 1.0L;
    }();
    for (int d : kDegrees) {
        const int n = d + 1;
        std::vector<long double> fv(n), c(n), mono(n, 0.0L), Tp(n, 0.0L), Tc(n, 0.0L);
        for (int j = 0; j < n; ++j) fv[j] = fq(std::cos(pi * (j + 0.5L) / n));
        for (int m = 0; m < n; ++m) {
            long double acc = 0.0L;
            for (int j = 0; j < n; ++j) acc += fv[j] * std::cos(pi * m * (j + 0.5L) / n);
            c[m] = 2.0L * acc / n;
        }
        c[0] /= 2.0L;
        // Chebyshev -> monomial: T_0 = 1, T_1 = t, T_{m+1} = 2 t T_m - T_{m-1}
        Tc[0] = 1.0L;
        for (int m = 0; m < n; ++m) {
            for (int i = 0; i <= m; ++i) mono[i] += c[m] * Tc[i];
            std::vector<long double> nx(n, 0.0L);
            if (m == 0) {
                if (n > 1) nx[1] = 1.0L;
            } else {
                for (int i = 0; i + 1 < n; ++i) nx[i + 1] += 2.0L * Tc[i];
                for (int i = 0; i < n; ++i) nx[i] -= Tp[i];
            }
            Tp = Tc;
            Tc = nx;
        }
        long double err = 0.0L;
        for (int k = 0; k <= 512; ++k) {
            const long double t = -1.0L + 2.0L * k / 512.0L;
            long double p = mono[d];
            for (int i = d - 1; i >= 0; --i) p = p * t + mono[i];
            err = std::max(err, std::fabs(p - fq(t)));
        }
        if (err <= qtol * tscale) {
            for (int i = 0; i < 33; ++i) pc[i] = i < n ? (double)mono[i] : 0.0;
            return d;
        }
    }
    return 0;
}

}  // namespace se

// ======================================================================
// extern "C" planning entry points
// ======================================================================
using namespace se;

#define SE_API_BEGIN try {
#define SE_API_END                                   \
    return SE_OK;                                    \
    }                                                \
    catch (const se::Error &e) {                     \
        se::set_last_error(e.what());                \
        return e.code;                               \
    }                                                \
    catch (const std::exception &e) {                \
        se::set_last_error(e.what());                \
        return SE_EDEVICE;                           \
    }

extern "C" {

const char *se_last_error(void) { return g_last_error.c_str(); }
const char *se_version(void) { return "se_b200 0.1 (sm_100a)"; }

int se_params_validate(const se_params_t *p, double L, int D) {
    SE_API_BEGIN
    if (!p) fail(SE_EINVAL, "null params");
    validate(*p, L, D);
    SE_API_END
}

int se_grid_build(int D, double L, const se_params_t *p, se_grid_t *out) {
    SE_API_BEGIN
    if (!p || !out) fail(SE_EINVAL, "null argument");
    if (D < 0 || D > 3) fail(SE_EINVAL, "D must be in {0,1,2,3}");
    *out = build_grid(D, L, *p);
    SE_API_END
}

int se_padded_size(double s, int32_t n, int32_t *out) {
    SE_API_BEGIN
    *out = padded_size(s, n);
    SE_API_END
}

int se_next_even_smooth(int32_t n, int32_t *out) {
    SE_API_BEGIN
    *out = next_even_smooth(n);
    SE_API_END
}

int se_pair_poly_coefficients(double xi, double rc, int kind, double *coeffs, int32_t *degree) {
    SE_API_BEGIN
    if (!coeffs || !degree) fail(SE_EINVAL, "null argument");
    if (!(xi > 0) || !(rc > 0)) fail(SE_EINVAL, "xi and rc must be positive");
    if (kind != 0 && kind != 1) fail(SE_EINVAL, "kind must be 0 (potential) or 1 (field)");
    *degree = pair_poly_fit(xi, rc, kind, coeffs);
    SE_API_END
}

int se_d0_kernel_geometry(double L, int32_t M, int32_t P, double s0, double rc, int32_t *nconv,
                          int32_t *g0, double *R) {
    SE_API_BEGIN
    D0Geom d = d0_geometry(L, M, P, s0, rc, !std::isnan(rc));
    *nconv = d.nconv;
    *g0 = d.g0;
    *R = d.R;
    SE_API_END
}

int se_mode_partition_counts(int32_t M, int D, int32_t nI, int64_t *nI_rows, int64_t *nJ_rows) {
    SE_API_BEGIN
    if (D != 1 && D != 2) fail(SE_EINVAL, "mode partitions apply to D in {1,2}");
    if (nI < 0 || nI > M / 2) fail(SE_EINVAL, "nI must lie in [0, M/2]");
    std::vector<int> m = signed_modes(M);
    int64_t ni = 0, nj = 0;
    for (int i = 0; i < M; ++i) {
        for (int j = 0; j < (D == 2 ? M : 1); ++j) {
            int mu = std::abs(m[i]);
            if (D == 2) mu = std::max(mu, std::abs(m[j]));
            if (mu >= 1 && mu <= nI) ++ni;
            if (mu > nI) ++nj;
        }
    }
    *nI_rows = ni;
    *nJ_rows = nj;
    SE_API_END
}

int se_window_eval(int window, int32_t P, double h, double shape, const double *x, int64_t n, double *out) {
    SE_API_BEGIN
    if (window < 0 || window > 2) fail(SE_EINVAL, "unknown window kind");
    if (P < 1 || !(h > 0) || !(shape > 0)) fail(SE_EINVAL, "invalid window parameters");
    double w = 0.5 * P * h;
    for (int64_t i = 0; i < n; ++i) out[i] = window_value(window, w, shape, x[i]);
    SE_API_END
}

int se_window_fourier(int window, int32_t P, double h, double shape, const double *k, int64_t n, double *out) {
    SE_API_BEGIN
    if (window < 0 || window > 2) fail(SE_EINVAL, "unknown window kind");
    if (P < 1 || !(h > 0) || !(shape > 0)) fail(SE_EINVAL, "invalid window parameters");
    std::vector<double> kv(k, k + n);
    std::vector<double> v = window_fourier(window, P, h, shape, kv);
    std::memcpy(out, v.data(), sizeof(double) * n);
    SE_API_END
}

int se_bm_quadrature(double w, double beta, const double *k, int64_t n, int32_t nodes, double *out) {
    SE_API_BEGIN
    if (!(w > 0) || !(beta >= 0) || nodes < 2) fail(SE_EINVAL, "invalid BM quadrature parameters");
    std::vector<double> kv(k, k + n);
    std::vector<double> v = bm_quadrature(w, beta, kv, nodes);
    std::memcpy(out, v.data(), sizeof(double) * n);
    SE_API_END
}

// realspace.py:43-59: bucket particles into n^3 cells of edge L/n, members of
// each cell in ascending index order (a stable counting sort).
int se_cell_list_host(const double *pos, int64_t N, double L, int32_t n, int64_t *order, int64_t *bounds) {
    SE_API_BEGIN
    if (n < 1 || !(L > 0)) fail(SE_EINVAL, "invalid cell list geometry");
    const int64_t nc = (int64_t)n * n * n;
    const double edge = L / n;
    std::vector<int64_t> cell(N);
    for (int64_t c = 0; c <= nc; ++c) bounds[c] = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t f = 0;
        for (int a = 0; a < 3; ++a) {
            int64_t c = (int64_t)(pos[3 * i + a] / edge);
            if (c > n - 1) c = n - 1;
            if (c < 0) c = 0;
            f = f * n + c;
        }
        cell[i] = f;
        bounds[f + 1]++;
    }
    for (int64_t c = 0; c < nc; ++c) bounds[c + 1] += bounds[c];
    std::vector<int64_t> fill(bounds, bounds + nc);
    for (int64_t i = 0; i < N; ++i) order[fill[cell[i]]++] = i;
    SE_API_END
}

int se_kb_sinhc(const double *rho2, int64_t n, double *out) {
    SE_API_BEGIN
    for (int64_t i = 0; i < n; ++i) out[i] = kb_sinhc(rho2[i]);
    SE_API_END
}

int se_greens_zero_mode(int D, double R, const double *kappa, int64_t n, double *out) {
    SE_API_BEGIN
    if (D < 0 || D > 2) fail(SE_EINVAL, "zero-mode kernel is defined for D < 3");
    for (int64_t i = 0; i < n; ++i) out[i] = greens_zero_mode(D, R, kappa[i]);
    SE_API_END
}

}  // extern "C"
