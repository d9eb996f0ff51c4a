// extern "C" entry points of the SE B200 library (include/se_b200.h):
// plan lifetime, stage calls on device pointers, fused pipelines
// (se_kspace / total_potential), sharded variants and host-buffer variants.
#include <cstring>

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

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        SE_CUDA(cudaGetDevice(&prev));
        if (prev != dev) SE_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

se_plan *checked(se_plan_t p) {
    if (!p) fail(SE_EINVAL, "null plan");
    return p;
}

size_t grid_points(const se_plan *pl) { return (size_t)pl->g.shape[0] * pl->g.shape[1] * pl->g.shape[2]; }

// charge sums and box check in one pass: [sum q, sum |q|, #outside [0,L)]
__global__ void check_kernel(const double *__restrict__ pos, const double *__restrict__ q, int64_t N, double L,
                             double *__restrict__ out) {
    double s = 0.0, a = 0.0, bad = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (q) {
            const double qi = q[i];
            s += qi;
            a += fabs(qi);
        }
        for (int ax = 0; ax < 3; ++ax) {
            double x = pos[3 * i + ax];
            if (!(x >= 0.0 && x < L)) bad += 1.0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        a += __shfl_xor_sync(0xffffffffu, a, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    // block reduction, then one atomic per block and quantity (per-warp
    // atomics on three addresses serialise: ~50 us at N = 1e6)
    __shared__ double red[3][32];
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = s;
        red[1][w] = a;
        red[2][w] = bad;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double v = 0.0;
        for (int i = 0; i < nw; ++i) v += red[threadIdx.x][i];
        atomicAdd(out + threadIdx.x, v);
    }
}

// core.py:65-77 (box) and core.py:180-191 (neutrality): ValueError for D > 0,
// a warning flag for D = 0.
// the check kernel alone (no host synchronisation; capturable)
void check_launch(se_plan *pl, const double *pos, const double *q, int64_t N) {
    SE_CUDA(cudaMemsetAsync(pl->check.ptr, 0, sizeof(double) * 4, pl->stream));
    int64_t blocks = (N + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    check_kernel<<<(unsigned)blocks, 256, 0, pl->stream>>>(pos, q, N, pl->L, pl->check.as<double>());
    SE_LAUNCH_CHECK();
    pl->launches += 1;
}

// the verdict on the check kernel's sums h = [sum q, sum |q|, #outside]
void check_verdict(se_plan *pl, const double *h, bool neutrality) {
    if (h[2] > 0) fail(SE_EINVAL, "all coordinates must lie in [0, L)");
    if (!neutrality) return;
    double qabs = h[1] > 1.0 ? h[1] : 1.0;
    if (std::fabs(h[0]) <= 1e-12 * qabs) return;
    if (pl->D == 0)
        pl->warnings |= 1;
    else
        fail(SE_EINVAL, "periodic Ewald summation requires a charge-neutral system");
}

void check_system(se_plan *pl, const double *pos, const double *q, int64_t N, bool neutrality) {
    pl->warnings = 0;
    if (N <= 0) return;
    pl->check.ensure(sizeof(double) * 4);
    check_launch(pl, pos, q, N);
    double h[4];
    SE_CUDA(cudaMemcpyAsync(h, pl->check.ptr, sizeof(double) * 4, cudaMemcpyDeviceToHost, pl->stream));
    SE_CUDA(cudaStreamSynchronize(pl->stream));
    check_verdict(pl, h, neutrality);
}

void flag_verdict(int h) {
    if (h == 1) fail(SE_ESINGULAR, "coincident distinct particles");
    if (h == 2) fail(SE_ESINGULAR, "particle coincides with an image");
}

void check_flag(se_plan *pl) {
    int h = 0;
    SE_CUDA(cudaMemcpyAsync(&h, pl->flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, pl->stream));
    SE_CUDA(cudaStreamSynchronize(pl->stream));
    flag_verdict(h);
}

// The fused total potential checks its input WITHOUT a host round trip
// before the device work: the check kernel is the first node of the body
// (inside the CUDA graph), the binning kernels read coordinates through
// sane_coord (se_common.h) so invalid input cannot index out of range, and
// the sums come back together with the singularity flag (and, for the
// _host entry, the potentials) under ONE synchronisation at the end.  The
// caller sees the reference's errors in the reference's order (box,
// neutrality, coincidence); only their timing moved (the timeline of
// profiles/timeline_cfg2_r02.txt: 0.1 ms of idle GPU per call at cfg2).
void total_verdict(se_plan *pl, int64_t N, const void *extra_dev, void *extra_host, size_t extra_bytes) {
    if (!pl->verdict_host) SE_CUDA(cudaMallocHost((void **)&pl->verdict_host, sizeof(double) * 5));
    double *h = pl->verdict_host;
    int *f = reinterpret_cast<int *>(h + 4);
    *f = 0;
    const bool checked_run = N > 0 && pl->check.ptr && pl->flag.ptr;
    if (checked_run) {
        SE_CUDA(cudaMemcpyAsync(h, pl->check.ptr, sizeof(double) * 4, cudaMemcpyDeviceToHost, pl->stream));
        SE_CUDA(cudaMemcpyAsync(f, pl->flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, pl->stream));
    }
    if (extra_bytes)
        SE_CUDA(cudaMemcpyAsync(extra_host, extra_dev, extra_bytes, cudaMemcpyDeviceToHost, pl->stream));
    SE_CUDA(cudaStreamSynchronize(pl->stream));
    if (checked_run) {
        check_verdict(pl, h, true);
        flag_verdict(*f);
    }
}

struct Events {
    bool on;
    cudaStream_t st;
    cudaEvent_t e[6];
    int n = 0;
    Events(bool enabled, cudaStream_t s) : on(enabled), st(s) {
        if (on)
            for (auto &x : e) SE_CUDA(cudaEventCreate(&x));
    }
    void mark() {
        if (on) SE_CUDA(cudaEventRecord(e[n++], st));
    }
    double secs(int a, int b) {
        float ms = 0;
        SE_CUDA(cudaEventElapsedTime(&ms, e[a], e[b]));
        return ms * 1e-3;
    }
    ~Events() {
        if (on)
            for (auto &x : e) cudaEventDestroy(x);
    }
};

// spread -> k-space -> gather (sekspace.py:340-389); phi += or = phi_F
void kspace_pipeline(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi, int use_kernel,
                     double *timings, int accumulate, int rank, int world, bool capturing = false) {
    double *grid = nullptr;
    pl->grid_dev.ensure(sizeof(double) * grid_points(pl));
    grid = pl->grid_dev.as<double>();
    Events ev(timings != nullptr, pl->stream);
    ev.mark();
    spread_run(pl, pos, q, N, grid, 0, 1);  // every rank needs the full grid; see the shard API for splitting
    ev.mark();
    double kt[SE_T_COUNT] = {0};
    prof_begin(pl, SE_K_KSPACE);
    kspace_run(pl, grid, use_kernel, timings ? kt : nullptr);
    prof_end(pl, SE_K_KSPACE);
    ev.mark();
    gather_run(pl, grid, pos, N, phi, accumulate, rank, world, false);
    ev.mark();
    if (!capturing) prof_collect(pl);
    if (timings) {
        SE_CUDA(cudaStreamSynchronize(pl->stream));
        timings[SE_T_SPREAD] = ev.secs(0, 1);
        timings[SE_T_AFT] = kt[SE_T_AFT];
        timings[SE_T_SCALE] = kt[SE_T_SCALE];
        timings[SE_T_AIFT] = kt[SE_T_AIFT];
        timings[SE_T_PRECOMPUTE] = kt[SE_T_PRECOMPUTE];
        timings[SE_T_GATHER] = ev.secs(2, 3);
    }
}

void graph_drop(se_plan *pl) {
    if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
    pl->gexec = nullptr;
    pl->gwarm = false;
    pl->gN = -1;
}

__global__ void add_kernel(double *__restrict__ phi, const double *__restrict__ add, int64_t N) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) phi[i] += add[i];
}

// The device work of total_potential after validation: no host syncs, so
// it can be captured into a CUDA graph.  The k-space pipeline (spread ->
// FFT / multiplier -> gather, shared-memory / LSU bound) runs on a
// higher-priority side stream concurrently with the real-space kernel
// (issue / fp64 bound) and lands in its own buffer; phi_R + self is written
// by the real-space finish, then phi += phi_F after the join.
void total_body(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi, bool capturing) {
    if (!pl->side) {
        int lo = 0, hi = 0;
        SE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        SE_CUDA(cudaStreamCreateWithPriority(&pl->side, cudaStreamNonBlocking, hi));
        SE_CUDA(cudaEventCreateWithFlags(&pl->fork_ev, cudaEventDisableTiming));
        SE_CUDA(cudaEventCreateWithFlags(&pl->join_ev, cudaEventDisableTiming));
    }
    pl->phik.ensure(sizeof(double) * (N ? N : 1));
    cudaStream_t main_st = pl->stream;
    check_launch(pl, pos, q, N);  // read back by total_verdict
    SE_CUDA(cudaEventRecord(pl->fork_ev, main_st));
    SE_CUDA(cudaStreamWaitEvent(pl->side, pl->fork_ev, 0));
    pl->stream = pl->side;
    try {
        kspace_pipeline(pl, pos, q, N, pl->phik.as<double>(), 1, nullptr, 0, 0, 1, capturing);
    } catch (...) {
        pl->stream = main_st;
        throw;
    }
    pl->stream = main_st;
    SE_CUDA(cudaEventRecord(pl->join_ev, pl->side));
    realspace_run(pl, pos, q, N, phi, 1, 0, 1);
    SE_CUDA(cudaStreamWaitEvent(main_st, pl->join_ev, 0));
    add_kernel<<<(unsigned)((N + 255) / 256), 256, 0, main_st>>>(phi, pl->phik.as<double>(), N);
    SE_LAUNCH_CHECK();
    pl->launches += 1;
}

// Repeated calls with the same (pos, q, phi, N, stream) replay a CUDA graph
// of the body: the first call runs it eagerly (allocating every buffer and
// table), the second captures and instantiates it, later ones launch the
// graph -- ~40 kernel / memset / FFT launches become one.  The legacy default
// stream cannot be captured: the graph then runs on the plan's own stream,
// fenced after and before the caller's stream by events.
void graph_capture(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi) {
    const int64_t l0 = pl->launches;
    bool pend0[SE_K_COUNT];
    for (int id = 0; id < SE_K_COUNT; ++id) pend0[id] = pl->pending[id];
    cudaGraph_t graph = nullptr;
    SE_CUDA(cudaStreamBeginCapture(pl->stream, cudaStreamCaptureModeRelaxed));
    pl->capturing = true;
    try {
        total_body(pl, pos, q, N, phi, true);
    } catch (...) {
        pl->capturing = false;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(pl->stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    pl->capturing = false;
    SE_CUDA(cudaStreamEndCapture(pl->stream, &graph));
    cudaError_t e = cudaGraphInstantiate(&pl->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        pl->gexec = nullptr;
        SE_CUDA(e);
    }
    pl->glaunches = pl->launches - l0;
    for (int id = 0; id < SE_K_COUNT; ++id) pl->gpending[id] = pl->pending[id] && !pend0[id];
}

void total_body_graphed(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi) {
    const bool same = pl->gN == N && pl->gkey[0] == pos && pl->gkey[1] == q && pl->gkey[2] == phi &&
                      pl->gstream == pl->stream && pl->gprof == pl->prof &&
                      pl->ggen == g_buf_generation.load();
    if (!same || !pl->gwarm) {
        graph_drop(pl);
        total_body(pl, pos, q, N, phi, false);
        pl->gkey[0] = pos;
        pl->gkey[1] = q;
        pl->gkey[2] = phi;
        pl->gN = N;
        pl->gstream = pl->stream;
        pl->gprof = pl->prof;
        pl->ggen = g_buf_generation.load();
        pl->gwarm = true;
        return;
    }
    cudaStream_t user = pl->stream;
    const bool legacy = user == nullptr || user == cudaStreamLegacy || user == cudaStreamPerThread;
    cudaStream_t gs = legacy ? pl->own_stream : user;
    if (legacy) {
        for (auto &ev : pl->gfence)
            if (!ev) SE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        SE_CUDA(cudaEventRecord(pl->gfence[0], user));
        SE_CUDA(cudaStreamWaitEvent(gs, pl->gfence[0], 0));
    }
    if (!pl->gexec) {
        pl->stream = gs;
        try {
            graph_capture(pl, pos, q, N, phi);
        } catch (...) {
            pl->stream = user;
            graph_drop(pl);
            throw;
        }
        pl->stream = user;
        if (pl->ggen != g_buf_generation.load()) {  // the body allocated after all: do not keep it
            graph_drop(pl);
            if (legacy) {
                SE_CUDA(cudaEventRecord(pl->gfence[1], gs));
                SE_CUDA(cudaStreamWaitEvent(user, pl->gfence[1], 0));
            }
            total_body(pl, pos, q, N, phi, false);
            return;
        }
    } else {
        pl->launches += pl->glaunches;
        for (int id = 0; id < SE_K_COUNT; ++id)
            if (pl->gpending[id]) pl->pending[id] = true;
    }
    SE_CUDA(cudaGraphLaunch(pl->gexec, gs));
    if (legacy) {
        SE_CUDA(cudaEventRecord(pl->gfence[1], gs));
        SE_CUDA(cudaStreamWaitEvent(user, pl->gfence[1], 0));
    }
}

template <class T>
T *stage_in(se_plan *pl, DevBuf &b, const T *host, size_t n) {
    b.ensure(sizeof(T) * (n ? n : 1));
    if (n) SE_CUDA(cudaMemcpyAsync(b.ptr, host, sizeof(T) * n, cudaMemcpyHostToDevice, pl->stream));
    return b.as<T>();
}

void stage_out(se_plan *pl, void *host, const void *dev, size_t bytes) {
    if (bytes) SE_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, pl->stream));
    SE_CUDA(cudaStreamSynchronize(pl->stream));
}

void total_pipeline(se_plan *pl, const double *pos, const double *q, int64_t N, double *phi, double *timings,
                    void *out_host = nullptr) {
    if (!timings && N > 0) {
        pl->warnings = 0;
        pl->check.ensure(sizeof(double) * 4);
        if (pl->graphs)
            total_body_graphed(pl, pos, q, N, phi);
        else
            total_body(pl, pos, q, N, phi, false);
        total_verdict(pl, N, phi, out_host, out_host ? sizeof(double) * N : 0);
    } else {
        check_system(pl, pos, q, N, true);
        Events ev(timings != nullptr, pl->stream);
        ev.mark();
        realspace_run(pl, pos, q, N, phi, 1, 0, 1);
        ev.mark();
        kspace_pipeline(pl, pos, q, N, phi, 1, timings, 1, 0, 1);
        if (timings) timings[SE_T_REALSPACE] = ev.secs(0, 1);
        check_flag(pl);
        if (out_host) stage_out(pl, out_host, phi, sizeof(double) * N);
    }
    prof_collect(pl);
}

// realspace.py:183-185: -2 xi q / sqrt(pi)
__global__ void self_kernel(const double *__restrict__ q, int64_t N, double xi, double sqrtpi, double *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) out[i] = (-2.0 * xi * q[i]) / sqrtpi;
}

void check_shard(int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) fail(SE_EINVAL, "invalid shard (rank, world)");
}

}  // namespace

namespace se {
void plan_release_device(se_plan *pl) {
    if (pl->side) cudaStreamSynchronize(pl->side);
    if (pl->side) cudaStreamDestroy(pl->side);
    if (pl->fork_ev) cudaEventDestroy(pl->fork_ev);
    if (pl->join_ev) cudaEventDestroy(pl->join_ev);
    pl->phik.release();
    pl->fgrid.release();
    pl->fphi.release();
    pl->io_E.release();
    if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
    pl->gexec = nullptr;
    for (auto &ev : pl->gfence)
        if (ev) cudaEventDestroy(ev);
    for (cufftHandle h : {pl->fft_fwd, pl->fft_inv, pl->fft_rowJ, pl->fft_rowI, pl->fft_row0, pl->fft_c_fwd,
                          pl->fft_c_inv, pl->fft_f_fwd, pl->fft_f_inv, pl->slab_f2, pl->slab_i2, pl->slab_x,
                          pl->zs_fwd, pl->zs_inv, pl->zs_rowJ, pl->zs_rowI, pl->zs_row0})
        if (h) cufftDestroy(h);
    for (Binning *b : {&pl->tbin, &pl->cbin})
        for (DevBuf *d : {&b->keys, &b->keys_sorted, &b->idx, &b->idx_sorted, &b->counts, &b->starts, &b->units,
                          &b->nunits, &b->ubstart, &b->fhist, &b->fstart, &b->bsum, &b->large, &b->nlarge, &b->rec})
            d->release();
    for (ModeTable *t : {&pl->tM, &pl->tg0, &pl->tgs, &pl->tMt, &pl->tNc, &pl->tNh}) {
        t->k.release();
        t->what.release();
    }
    for (DevBuf *d : {&pl->flag, &pl->spec, &pl->spec2, &pl->spec3, &pl->work, &pl->grid_tmp, &pl->rows_I,
                      &pl->ghat, &pl->grid_dev, &pl->io_pos, &pl->io_q, &pl->io_phi, &pl->io_grid, &pl->check, &pl->pairs, &pl->racc, &pl->sdet,
                      &pl->zs_rowsI, &pl->zs_Hk, &pl->zs_Z, &pl->zs_B})
        d->release();
    if (pl->verdict_host) cudaFreeHost(pl->verdict_host);
    pl->verdict_host = nullptr;
    if (pl->own_stream) cudaStreamDestroy(pl->own_stream);
}
}  // namespace se

extern "C" {

int se_plan_create(se_plan_t *plan, int D, double L, const se_params_t *p, int device) {
    SE_API_BEGIN
    if (!plan || !p) fail(SE_EINVAL, "null argument");
    *plan = nullptr;
    validate(*p, L, D);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        fail(SE_EDEVICE, "no CUDA device available (the SE B200 library has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) fail(SE_EINVAL, "device ordinal out of range");
    DeviceGuard dg(device);
    se_plan *pl = new se_plan();
    pl->D = D;
    pl->L = L;
    pl->p = *p;
    pl->device = device;
    {
        const char *det = std::getenv("SE_B200_DETERMINISTIC");
        pl->deterministic = det && det[0] && det[0] != '0';
    }
    try {
        pl->g = build_grid(D, L, *p);
        SE_CUDA(cudaStreamCreateWithFlags(&pl->own_stream, cudaStreamNonBlocking));
        pl->stream = pl->own_stream;
    } catch (...) {
        delete pl;
        throw;
    }
    *plan = pl;
    SE_API_END
}

int se_plan_destroy(se_plan_t plan) {
    SE_API_BEGIN
    if (!plan) return SE_OK;
    {
        DeviceGuard dg(plan->device);
        cudaStreamSynchronize(plan->stream);
        plan_release_device(plan);
    }
    delete plan;
    SE_API_END
}

int se_plan_set_stream(se_plan_t plan, void *stream) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    pl->stream = (cudaStream_t)stream;  // 0 is the legacy default stream
    SE_API_END
}

int se_plan_set_deferred_checks(se_plan_t plan, int on) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    pl->defer = on != 0;
    SE_API_END
}

int se_plan_finish(se_plan_t plan) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    if (pl->flag.ptr) check_flag(pl);
    prof_collect(pl);
    SE_API_END
}

int se_plan_set_deterministic(se_plan_t plan, int on) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    pl->deterministic = on != 0;
    graph_drop(pl);
    SE_API_END
}

int se_plan_set_graphs(se_plan_t plan, int on) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    pl->graphs = on != 0;
    if (!pl->graphs) graph_drop(pl);
    SE_API_END
}

int se_plan_set_profiling(se_plan_t plan, int on) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    pl->prof = on != 0;
    for (int i = 0; i < SE_K_COUNT; ++i) {
        pl->pms[i] = 0.0;
        pl->pcount[i] = 0;
        pl->pending[i] = false;
    }
    SE_API_END
}

int se_plan_kernel_times(se_plan_t plan, double *ms, int64_t *launches) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    prof_collect(pl);
    for (int i = 0; i < SE_K_COUNT; ++i) {
        if (ms) ms[i] = pl->pms[i];
        if (launches) launches[i] = pl->pcount[i];
    }
    SE_API_END
}

int se_realspace_pair_count_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, int64_t *pairs) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    long long n = 0;
    realspace_pair_count(pl, pos, q, N, &n);
    *pairs = n;
    SE_API_END
}

int se_plan_grid(se_plan_t plan, se_grid_t *out) {
    SE_API_BEGIN
    *out = checked(plan)->g;
    SE_API_END
}

int se_plan_launch_count(se_plan_t plan, int64_t *count) {
    SE_API_BEGIN
    *count = checked(plan)->launches;
    SE_API_END
}

int se_plan_warnings(se_plan_t plan, int *flags) {
    SE_API_BEGIN
    *flags = checked(plan)->warnings;
    SE_API_END
}

int se_check_system_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, int neutrality) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    check_system(pl, pos, q, N, neutrality != 0 && q != nullptr);
    SE_API_END
}

int se_spread_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, double *grid_out) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    check_system(pl, pos, nullptr, N, false);
    spread_run(pl, pos, q, N, grid_out, 0, 1);
    SE_API_END
}

int se_spread_shard_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, int rank, int world,
                        double *grid_out) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    check_shard(rank, world);
    DeviceGuard dg(pl->device);
    if (!pl->defer) check_system(pl, pos, nullptr, N, false);
    spread_run(pl, pos, q, N, grid_out, rank, world);
    if (!pl->defer) prof_collect(pl);
    SE_API_END
}

int se_kspace_apply_dev(se_plan_t plan, double *grid, int use_kernel, double *timings) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    prof_begin(pl, SE_K_KSPACE);
    kspace_run(pl, grid, use_kernel, timings);
    prof_end(pl, SE_K_KSPACE);
    if (!pl->defer) prof_collect(pl);
    SE_API_END
}

int se_slab_geometry(se_plan_t plan, int world, int64_t *nx, int64_t *nky, int64_t *nkz) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    if (!nx || !nky || !nkz) fail(SE_EINVAL, "null output pointer");
    slab_geometry(pl, world, nx, nky, nkz);
    SE_API_END
}

int se_slab_forward_dev(se_plan_t plan, int world, const double *slab, double *send) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    slab_forward(pl, world, slab, send);
    SE_API_END
}

int se_slab_xpass_dev(se_plan_t plan, int world, int rank, double *recv) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    slab_xpass(pl, world, rank, recv);
    SE_API_END
}

int se_slab_inverse_dev(se_plan_t plan, int world, const double *back, double *slab) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    slab_inverse(pl, world, back, slab);
    SE_API_END
}

int se_zslab_geometry(se_plan_t plan, int world, int rank, int64_t *out6) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    if (!out6) fail(SE_EINVAL, "null output pointer");
    zslab_geometry(pl, world, rank, out6);
    SE_API_END
}

int se_zslab_forward_dev(se_plan_t plan, int world, int rank, const double *zslab, double *spec) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    zslab_forward(pl, world, rank, zslab, spec);
    SE_API_END
}

int se_zslab_rows_dev(se_plan_t plan, int world, int rank, double *recv) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    zslab_rows(pl, world, rank, recv);
    SE_API_END
}

int se_zslab_inverse_dev(se_plan_t plan, int world, int rank, const double *spec, double *zslab) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    zslab_inverse(pl, world, rank, spec, zslab);
    SE_API_END
}

int se_gather_dev(se_plan_t plan, const double *grid, const double *pos, int64_t N, double *phi, int accumulate) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    check_system(pl, pos, nullptr, N, false);
    gather_run(pl, grid, pos, N, phi, accumulate, 0, 1, true);
    SE_API_END
}

int se_gather_shard_dev(se_plan_t plan, const double *grid, const double *pos, int64_t N, int rank, int world,
                        double *phi, int accumulate) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    check_shard(rank, world);
    DeviceGuard dg(pl->device);
    if (!pl->defer) check_system(pl, pos, nullptr, N, false);
    gather_run(pl, grid, pos, N, phi, accumulate, rank, world, true);
    if (!pl->defer) prof_collect(pl);
    SE_API_END
}

int se_kspace_potential_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, double *phi, int use_kernel,
                            double *timings) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    check_system(pl, pos, nullptr, N, false);
    kspace_pipeline(pl, pos, q, N, phi, use_kernel, timings, 0, 0, 1);
    SE_API_END
}

int se_realspace_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, double *phi, int add_self) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    check_system(pl, pos, nullptr, N, false);
    realspace_run(pl, pos, q, N, phi, add_self, 0, 1);
    check_flag(pl);
    SE_API_END
}

int se_realspace_shard_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, int rank, int world,
                           double *phi, int add_self) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    check_shard(rank, world);
    DeviceGuard dg(pl->device);
    if (!pl->defer) check_system(pl, pos, nullptr, N, false);
    realspace_run(pl, pos, q, N, phi, add_self, rank, world);
    if (!pl->defer) {
        check_flag(pl);
        prof_collect(pl);
    }
    SE_API_END
}

int se_realspace_domain_dev(se_plan_t plan, const double *pos, const double *q, int64_t n_local, int64_t n_own,
                            int ncols, int col_lo, int col_hi, double *phi, int add_self) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    if (!pl->defer) check_system(pl, pos, nullptr, n_local, false);
    realspace_domain_run(pl, pos, q, n_local, n_own, ncols, col_lo, col_hi, phi, add_self);
    if (!pl->defer) {
        check_flag(pl);
        prof_collect(pl);
    }
    SE_API_END
}

int se_total_potential_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, double *phi,
                           double *timings) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    total_pipeline(pl, pos, q, N, phi, timings);
    SE_API_END
}

__global__ void field_combine_kernel(const double *__restrict__ ek, int64_t N, double *__restrict__ E) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    E[3 * i] += ek[i];
    E[3 * i + 1] += ek[N + i];
    E[3 * i + 2] += ek[2 * N + i];
}

// E = E_R + E_F at every particle (D = 3): the real-space field kernel, then
// spread -> scaled spectrum -> three differentiated inverse transforms ->
// three gathers, summed into E (N x 3, caller order).
// Fourier part of the field (D = 3): spread -> scaled spectrum -> three
// differentiated inverse transforms -> three gathers; E = E_F (accumulate
// 0) or E += E_F.
void kspace_field_pipeline(se_plan *pl, const double *pos, const double *q, int64_t N, double *E, int accumulate) {
    if (N <= 0) return;
    if (pl->D != 3) {
        // D < 3: the potential's k-space stage (AFT or the D = 0 kernel path),
        // then the gradient of the gather (window derivative; Gaussian / KB)
        if (pl->p.window == SE_WINDOW_BM)
            fail(SE_EINVAL, "forces for D < 3 need the Gaussian or Kaiser-Bessel window (the ES window's "
                            "derivative is singular at its support edge)");
        pl->grid_dev.ensure(sizeof(double) * grid_points(pl));
        double *grid = pl->grid_dev.as<double>();
        spread_run(pl, pos, q, N, grid, 0, 1);
        prof_begin(pl, SE_K_KSPACE);
        kspace_run(pl, grid, 1, nullptr);
        prof_end(pl, SE_K_KSPACE);
        grad_gather_run(pl, grid, pos, N, E, accumulate);
        return;
    }
    const size_t G = grid_points(pl);
    pl->grid_dev.ensure(sizeof(double) * G);
    pl->fgrid.ensure(sizeof(double) * 3 * G);
    pl->fphi.ensure(sizeof(double) * 3 * (size_t)N);
    double *grid = pl->grid_dev.as<double>();
    spread_run(pl, pos, q, N, grid, 0, 1);
    prof_begin(pl, SE_K_KSPACE);
    kspace_field_run(pl, grid, pl->fgrid.as<double>());
    prof_end(pl, SE_K_KSPACE);
    for (int a = 0; a < 3; ++a)
        gather_run(pl, pl->fgrid.as<double>() + a * G, pos, N, pl->fphi.as<double>() + a * N, 0, 0, 1, false);
    if (!accumulate) SE_CUDA(cudaMemsetAsync(E, 0, sizeof(double) * 3 * N, pl->stream));
    field_combine_kernel<<<(unsigned)((N + 255) / 256), 256, 0, pl->stream>>>(pl->fphi.as<double>(), N, E);
    SE_LAUNCH_CHECK();
    pl->launches += 1;
}

void field_pipeline(se_plan *pl, const double *pos, const double *q, int64_t N, double *E) {
    check_system(pl, pos, q, N, true);
    realspace_field_run(pl, pos, q, N, E, 0, 1);
    kspace_field_pipeline(pl, pos, q, N, E, 1);
    check_flag(pl);
    prof_collect(pl);
}

int se_realspace_field_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    const double *dq = stage_in(pl, pl->io_q, q, (size_t)N);
    pl->io_E.ensure(sizeof(double) * 3 * (N ? N : 1));
    realspace_field_run(pl, dp, dq, N, pl->io_E.as<double>(), 0, 1);
    check_flag(pl);
    stage_out(pl, E, pl->io_E.ptr, sizeof(double) * 3 * N);
    SE_API_END
}

int se_kspace_field_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    const double *dq = stage_in(pl, pl->io_q, q, (size_t)N);
    pl->io_E.ensure(sizeof(double) * 3 * (N ? N : 1));
    kspace_field_pipeline(pl, dp, dq, N, pl->io_E.as<double>(), 0);
    stage_out(pl, E, pl->io_E.ptr, sizeof(double) * 3 * N);
    SE_API_END
}

int se_total_field_dev(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    field_pipeline(pl, pos, q, N, E);
    SE_API_END
}

int se_total_field_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *E) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    const double *dq = stage_in(pl, pl->io_q, q, (size_t)N);
    pl->io_E.ensure(sizeof(double) * 3 * (N ? N : 1));
    field_pipeline(pl, dp, dq, N, pl->io_E.as<double>());
    stage_out(pl, E, pl->io_E.ptr, sizeof(double) * 3 * N);
    SE_API_END
}

int se_total_potential_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *phi,
                            double *timings) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    const double *dq = stage_in(pl, pl->io_q, q, (size_t)N);
    pl->io_phi.ensure(sizeof(double) * (N ? N : 1));
    total_pipeline(pl, dp, dq, N, pl->io_phi.as<double>(), timings, phi);
    SE_API_END
}

int se_kspace_potential_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *phi,
                             int use_kernel, double *timings) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    const double *dq = stage_in(pl, pl->io_q, q, (size_t)N);
    pl->io_phi.ensure(sizeof(double) * (N ? N : 1));
    kspace_pipeline(pl, dp, dq, N, pl->io_phi.as<double>(), use_kernel, timings, 0, 0, 1);
    stage_out(pl, phi, pl->io_phi.ptr, sizeof(double) * N);
    SE_API_END
}

int se_spread_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *grid_out) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    const double *dq = stage_in(pl, pl->io_q, q, (size_t)N);
    pl->io_grid.ensure(sizeof(double) * grid_points(pl));
    spread_run(pl, dp, dq, N, pl->io_grid.as<double>(), 0, 1);
    stage_out(pl, grid_out, pl->io_grid.ptr, sizeof(double) * grid_points(pl));
    SE_API_END
}

int se_gather_host(se_plan_t plan, const double *grid, const double *pos, int64_t N, double *phi) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dg_ = stage_in(pl, pl->io_grid, grid, grid_points(pl));
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    pl->io_phi.ensure(sizeof(double) * (N ? N : 1));
    gather_run(pl, dg_, dp, N, pl->io_phi.as<double>(), 0, 0, 1, true);
    stage_out(pl, phi, pl->io_phi.ptr, sizeof(double) * N);
    SE_API_END
}

int se_kspace_apply_host(se_plan_t plan, double *grid, int use_kernel) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    double *d = stage_in(pl, pl->io_grid, (const double *)grid, grid_points(pl));
    kspace_run(pl, d, use_kernel, nullptr);
    stage_out(pl, grid, d, sizeof(double) * grid_points(pl));
    SE_API_END
}

int se_realspace_host(se_plan_t plan, const double *pos, const double *q, int64_t N, double *phi, int add_self) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    DeviceGuard dg(pl->device);
    const double *dp = stage_in(pl, pl->io_pos, pos, 3 * (size_t)N);
    const double *dq = stage_in(pl, pl->io_q, q, (size_t)N);
    pl->io_phi.ensure(sizeof(double) * (N ? N : 1));
    realspace_run(pl, dp, dq, N, pl->io_phi.as<double>(), add_self, 0, 1);
    check_flag(pl);
    stage_out(pl, phi, pl->io_phi.ptr, sizeof(double) * N);
    SE_API_END
}

int se_d0_kernel_table_host(se_plan_t plan, double *out) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    if (pl->D != 0) fail(SE_EINVAL, "the truncated-kernel table exists for D = 0 only");
    DeviceGuard dg(pl->device);
    d0_kernel_prepare(pl, nullptr);
    size_t n = (size_t)pl->nconv * pl->nconv * (pl->nconv / 2 + 1);
    stage_out(pl, out, pl->ghat.ptr, sizeof(double) * n);
    SE_API_END
}

int se_plan_d0_geometry(se_plan_t plan, int32_t *nconv, int32_t *g0, double *R) {
    SE_API_BEGIN
    se_plan *pl = checked(plan);
    D0Geom d = d0_geometry(pl->g.L, pl->g.M, pl->g.P, pl->p.s0, pl->p.rc, true);
    *nconv = d.nconv;
    *g0 = d.g0;
    *R = d.R;
    SE_API_END
}

int se_self_term_dev(const double *q, int64_t N, double xi, double *out, void *stream) {
    SE_API_BEGIN
    if (N > 0) {
        self_kernel<<<(unsigned)((N + 255) / 256), 256, 0, (cudaStream_t)stream>>>(q, N, xi, std::sqrt(M_PI), out);
        SE_LAUNCH_CHECK();
    }
    SE_API_END
}

int se_self_term_host(const double *q, int64_t N, double xi, double *out) {
    SE_API_BEGIN
    if (N <= 0) return SE_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        fail(SE_EDEVICE, "no CUDA device available (the SE B200 library has no CPU fallback)");
    }
    double *d = nullptr;
    SE_CUDA(cudaMalloc(&d, sizeof(double) * 2 * N));
    SE_CUDA(cudaMemcpy(d, q, sizeof(double) * N, cudaMemcpyHostToDevice));
    self_kernel<<<(unsigned)((N + 255) / 256), 256>>>(d, N, xi, std::sqrt(M_PI), d + N);
    cudaError_t e = cudaMemcpy(out, d + N, sizeof(double) * N, cudaMemcpyDeviceToHost);
    cudaFree(d);
    SE_CUDA(e);
    SE_API_END
}

}  // extern "C"
