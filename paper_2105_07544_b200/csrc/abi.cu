// libmpkb200: host launchers and the extern "C" ABI declared in
// include/mpk_b200.h.  The cycle driver (mpk_cycle_run) is the native
// runtime of one restarted-GMRES cycle: it enqueues every kernel of the
// cycle on the caller's stream without synchronising; early exits are
// device-side (ctl->done), so the host reads back once per cycle.
#include <cuda_runtime.h>

#include <cmath>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "comm.cuh"
#include "fused_dcgs2.cuh"

using namespace mpk;

namespace {

thread_local std::string g_err;
unsigned long long g_launches = 0;   // kernels enqueued by this library
thread_local const char *g_last_cycle = "";   // kernel family of the last mpk_cycle_run

int fail(int code, const char *msg) {
    g_err = msg;
    return code;
}

int check_launch(const char *what) {
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_err = std::string(what) + ": " + cudaGetErrorString(e);
        return MPK_ELAUNCH;
    }
    return MPK_OK;
}

int sm_count_cached() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

constexpr int kMaxBlocksPerSm = 8;

int max_blocks() { return sm_count_cached() * kMaxBlocksPerSm; }

// Grid = min(tiles, SMs x resident CTAs) for a grid-stride kernel.
template <class K> int grid_for(K kernel, size_t smem, int64_t n) {
    static std::mutex mu;
    static std::map<std::pair<const void *, size_t>, int> occ;
    static std::map<const void *, size_t> attr;   // dynamic shared memory opted in per kernel (only raised)
    int per_sm;
    {
        std::lock_guard<std::mutex> lk(mu);
        size_t &have = attr[(const void *)kernel];
        if (smem > have) {
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            have = smem;
        }
        auto key = std::make_pair((const void *)kernel, smem);
        auto it = occ.find(key);
        if (it == occ.end()) {
            int o = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, kBlock, smem);
            if (o < 1) o = 1;
            if (o > kMaxBlocksPerSm) o = kMaxBlocksPerSm;
            occ[key] = o;
            per_sm = o;
        } else {
            per_sm = it->second;
        }
    }
    int64_t tiles = (n + kBlock - 1) / kBlock;
    int64_t cap = (int64_t)sm_count_cached() * per_sm;
    int64_t g = tiles < cap ? tiles : cap;
    return (int)(g < 1 ? 1 : g);
}

// reduction workspace layout
struct Ws {
    unsigned *counters;
    void *partials;
    float *partials_low;
    void *sums;
};
// also holds the persistent cycle's 3 phases x (m + 2) slots x 320 CTAs (m <= 511)
int64_t ws_partials_bytes() {
    const int64_t multi = (int64_t)max_blocks() * kStride * 8;
    const int64_t cycle = 3LL * (MPK_MAX_STEPS + 2) * kFMaxCtas * 8;
    return multi > cycle ? multi : cycle;
}
int64_t ws_low_bytes() { return (int64_t)max_blocks() * 2 * 4; }
Ws carve(void *base) {
    char *p = (char *)base;
    Ws w;
    w.counters = (unsigned *)p;
    p += 256;
    w.partials = p;
    p += align_up(ws_partials_bytes(), 256);
    w.partials_low = (float *)p;
    p += align_up(ws_low_bytes(), 256);
    w.sums = p;
    return w;
}

// ---------------------------------------------------------------------------
// profiling: optional per-class CUDA events around cycle kernels
// ---------------------------------------------------------------------------
constexpr int kProfClasses = 8;
struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    double bytes;
};
std::vector<ProfRec> g_prof_live;
std::vector<cudaEvent_t> g_ev_pool;
double g_prof_ms[kProfClasses];
int64_t g_prof_cnt[kProfClasses];
double g_prof_bytes[kProfClasses];
bool g_prof_on = false;

cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_drain(bool wait) {
    size_t keep = 0;
    for (size_t i = 0; i < g_prof_live.size(); ++i) {
        ProfRec &r = g_prof_live[i];
        if (!wait && cudaEventQuery(r.b) != cudaSuccess) {
            g_prof_live[keep++] = r;
            continue;
        }
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        g_prof_ms[r.cls] += ms;
        g_prof_cnt[r.cls] += 1;
        g_prof_bytes[r.cls] += r.bytes;
        g_ev_pool.push_back(r.a);
        g_ev_pool.push_back(r.b);
    }
    g_prof_live.resize(keep);
}

struct ProfScope {
    bool on;
    ProfRec rec;
    cudaStream_t s;
    ProfScope(int cls, double bytes, cudaStream_t st) : on(g_prof_on), s(st) {
        if (!on) return;
        if (g_prof_live.size() > 8192) prof_drain(false);
        rec.a = ev_get();
        rec.b = ev_get();
        rec.cls = cls;
        rec.bytes = bytes;
        cudaEventRecord(rec.a, s);
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecord(rec.b, s);
        g_prof_live.push_back(rec);
    }
};

// ---------------------------------------------------------------------------
// operators
// ---------------------------------------------------------------------------
StencilConsts stencil_consts(const mpk_matrix *A) {
    StencilConsts k;
    memset(&k, 0, sizeof(k));
    k.preset = A->preset;
    k.nx = A->nx;
    k.row0 = A->row0;
    const double nx = (double)A->nx;
    k.nglob = (A->preset == MPK_LAPLACE3D) ? (int64_t)A->nx * A->nx * A->nx : (int64_t)A->nx * A->nx;
    volatile double h = 1.0 / (nx + 1.0);   // stencils.py:87
    k.h = h;
    k.dnx.init((uint32_t)A->nx);
    k.dnxy.init((uint32_t)A->nx * (uint32_t)A->nx);
    switch (A->preset) {
    case MPK_LAPLACE2D: {
        const double c[5] = {-1.0, -1.0, 4.0, -1.0, -1.0};
        memcpy(k.c, c, sizeof(c));
        break;
    }
    case MPK_LAPLACE3D: {
        const double c[7] = {-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0};
        memcpy(k.c, c, sizeof(c));
        break;
    }
    case MPK_UNIFLOW2D: {   // stencils.py:91-103
        volatile double d = A->diffusion;
        volatile double v = A->velocity / std::sqrt(2.0);
        volatile double hh = 0.5 * h;
        volatile double hv = hh * v;
        k.c[0] = -d - hv;
        k.c[1] = -d - hv;
        k.c[2] = 4.0 * d;
        k.c[3] = -d + hv;
        k.c[4] = -d + hv;
        break;
    }
    case MPK_BENTPIPE2D: {  // stencils.py:104-115 (per-row parts on device)
        volatile double c = A->convection;
        k.cc2 = c * 2.0;
        volatile double nc = -c;
        k.ncc2 = nc * 2.0;
        k.hh = 0.5 * h;
        k.c[2] = 4.0;
        break;
    }
    case MPK_STRETCHED2D: { // stencils.py:162-169
        volatile double a = 1.0 / A->stretch;
        volatile double b = A->stretch;
        volatile double ab = a + b;
        volatile double corner = -ab / 2.0;
        volatile double ew = b - 2.0 * a;
        volatile double ns = a - 2.0 * b;
        const double c[9] = {corner, ns, corner, ew, 4.0 * ab, ew, corner, ns, corner};
        memcpy(k.c, c, sizeof(c));
        break;
    }
    default:
        break;
    }
    return k;
}

template <typename T> StencilOp<T> make_stencil(const mpk_matrix *A) {
    StencilOp<T> op;
    op.n = A->n;
    op.k = stencil_consts(A);
    for (int i = 0; i < 9; ++i) op.cT[i] = (T)op.k.c[i];   // astype: round to nearest
    return op;
}

template <typename T> CsrOp<T> make_csr(const mpk_matrix *A) {
    CsrOp<T> op;
    op.n = A->n;
    op.rp = A->row_ptr;
    op.ci = A->col_idx;
    op.v = (const T *)A->values;
    op.band = (A->band > 0 && A->row0 == 0) ? A->band : 0;   // windows only on whole (one-GPU) matrices
    op.nnz_ = A->nnz;
    return op;
}

// Shared-memory x window of a banded CSR chunk: `rows` + 2*band elements,
// or 0 when the rows are short (<= 16 entries on average: their gathers hit
// L1, and the window costs occupancy -- C2's 5-entry rows ran 1.8x slower
// with it), the matrix is not banded, or the window would not fit.
constexpr int64_t kWinMaxBytes = 96 * 1024;
template <typename T> int64_t csr_window_elems(const CsrOp<T> &op, int64_t rows) {
    if (op.band <= 0 || op.n <= 0) return 0;
    if ((int64_t)op.nnz_ <= 16 * op.n) return 0;
    const int64_t e = rows + 2 * op.band;
    return e * (int64_t)sizeof(T) <= kWinMaxBytes ? e : 0;
}

// Two descriptors of the same operator (the polynomial's matrix and the
// cycle's): same kind, size, and storage or stencil definition.
bool same_operator(const mpk_matrix *a, const mpk_matrix *b) {
    if (a == b) return true;
    if (a->kind != b->kind || a->dtype != b->dtype || a->n != b->n || a->row0 != b->row0) return false;
    if (a->kind == MPK_CSR) return a->row_ptr == b->row_ptr && a->col_idx == b->col_idx && a->values == b->values;
    return a->preset == b->preset && a->nx == b->nx && a->diffusion == b->diffusion && a->velocity == b->velocity &&
           a->convection == b->convection && a->stretch == b->stretch;
}

template <typename T, class F> int with_op(const mpk_matrix *A, F &&f) {
    if (A->kind == MPK_STENCIL) return f(make_stencil<T>(A));
    if (A->kind == MPK_CSR) return f(make_csr<T>(A));
    return fail(MPK_EARG, "unknown matrix kind");
}

double spmv_bytes(const mpk_matrix *A, int sv) {
    // CSR: sv*(nnz + 2n) + 4*(nnz + n + 1); stencil: x read + y write
    if (A->kind == MPK_CSR) return (double)sv * (A->nnz + 2.0 * A->n) + 4.0 * (A->nnz + A->n + 1);
    return 2.0 * sv * A->n;
}

template <typename T> Hess<T> hess_view(void *base, int m) {
    Hess<T> H;
    T *p = (T *)base;
    H.m = m;
    H.h = p;
    p += (int64_t)(m + 1) * m;
    H.cs = p;
    p += m;
    H.sn = p;
    p += m;
    H.g = p;
    p += m + 1;
    H.d = p;
    p += m;
    H.raw = p;
    return H;
}

// ---------------------------------------------------------------------------
// pass launchers
// ---------------------------------------------------------------------------
template <typename T, int NC, class Op, bool NORM>
int launch_p1_nc(const Op &op, const T *src, const T *divp, T *vcol, const T *V, int64_t ld, int ndot, T *w,
                 Ws ws, T *out, T *out_wn2, const int32_t *done, cudaStream_t s) {
    auto kern = k_spmv_dot<T, NC, Op, NORM>;
    int g = grid_for(kern, 0, op.n);
    kern<<<g, kBlock, 0, s>>>(op, src, divp, vcol, V, ld, ndot, w, (T *)ws.partials, ws.counters, out,
                              out_wn2, done);
    return check_launch("k_spmv_dot");
}

template <typename T, class Op, bool NORM>
int launch_p1(const Op &op, const T *src, const T *divp, T *vcol, const T *V, int64_t ld, int ndot, T *w, Ws ws,
              T *out, T *out_wn2, const int32_t *done, cudaStream_t s) {
    if (ndot <= 8) return launch_p1_nc<T, 8, Op, NORM>(op, src, divp, vcol, V, ld, ndot, w, ws, out, out_wn2, done, s);
    if (ndot <= 16) return launch_p1_nc<T, 16, Op, NORM>(op, src, divp, vcol, V, ld, ndot, w, ws, out, out_wn2, done, s);
    if (ndot <= 32) return launch_p1_nc<T, 32, Op, NORM>(op, src, divp, vcol, V, ld, ndot, w, ws, out, out_wn2, done, s);
    return launch_p1_nc<T, kMaxCols, Op, NORM>(op, src, divp, vcol, V, ld, ndot, w, ws, out, out_wn2, done, s);
}

template <typename T, int NC>
int launch_multidot_nc(int64_t n, const T *V, int64_t ld, int ncols, const T *w, Ws ws, T *out,
                       const int32_t *done, cudaStream_t s) {
    auto kern = k_multidot<T, NC>;
    int g = grid_for(kern, 0, n);
    kern<<<g, kBlock, 0, s>>>(n, V, ld, ncols, w, (T *)ws.partials, ws.counters, out, done);
    return check_launch("k_multidot");
}

// out[c] = V[:, c]^T w for c < ncols, chunked by kMaxCols; writes out[ncols]
// = w.w of the last chunk's extra slot only when ncols <= kMaxCols.
template <typename T>
int launch_multidot(int64_t n, const T *V, int64_t ld, int ncols, const T *w, Ws ws, T *out,
                    const int32_t *done, cudaStream_t s) {
    for (int c0 = 0; c0 < ncols; c0 += kMaxCols) {
        int nc = ncols - c0 < kMaxCols ? ncols - c0 : kMaxCols;
        int rc;
        // scratch output so a chunk's extra slot never clobbers the next chunk
        T *dst = ((T *)ws.sums) + S_TMP;
        if (nc <= 8) rc = launch_multidot_nc<T, 8>(n, V + c0 * ld, ld, nc, w, ws, dst, done, s);
        else if (nc <= 16) rc = launch_multidot_nc<T, 16>(n, V + c0 * ld, ld, nc, w, ws, dst, done, s);
        else if (nc <= 32) rc = launch_multidot_nc<T, 32>(n, V + c0 * ld, ld, nc, w, ws, dst, done, s);
        else rc = launch_multidot_nc<T, kMaxCols>(n, V + c0 * ld, ld, nc, w, ws, dst, done, s);
        if (rc) return rc;
        cudaMemcpyAsync(out + c0, dst, sizeof(T) * nc, cudaMemcpyDeviceToDevice, s);
    }
    return MPK_OK;
}

template <typename T, int NC>
int launch_p2_nc(int64_t n, const T *V, int64_t ld, int ncols, const T *coef, const T *w, T *wout, Ws ws,
                 T *out, const int32_t *done, cudaStream_t s) {
    auto kern = k_update_dot<T, NC>;
    size_t smem = (size_t)ncols * kBlock * sizeof(T);
    int g = grid_for(kern, (size_t)NC * kBlock * sizeof(T), n);
    kern<<<g, kBlock, smem, s>>>(n, V, ld, ncols, coef, w, wout, (T *)ws.partials, ws.counters, out, done);
    return check_launch("k_update_dot");
}

template <typename T>
int launch_p2(int64_t n, const T *V, int64_t ld, int ncols, const T *coef, const T *w, T *wout, Ws ws,
              T *out, const int32_t *done, cudaStream_t s) {
    if (ncols <= 8) return launch_p2_nc<T, 8>(n, V, ld, ncols, coef, w, wout, ws, out, done, s);
    if (ncols <= 16) return launch_p2_nc<T, 16>(n, V, ld, ncols, coef, w, wout, ws, out, done, s);
    if (ncols <= 32) return launch_p2_nc<T, 32>(n, V, ld, ncols, coef, w, wout, ws, out, done, s);
    return launch_p2_nc<T, kMaxCols>(n, V, ld, ncols, coef, w, wout, ws, out, done, s);
}

template <typename T>
int launch_p3(int64_t n, const T *V, int64_t ld, int ncols, const T *coef, const T *w, T *wout, Ws ws,
              Hess<T> H, mpk_cycle_ctl *ctl, StepParams p, int do_givens, const int32_t *done,
              cudaStream_t s) {
    auto kern = k_update_norm<T>;
    int m = H.m > 0 ? H.m : 0;
    int64_t elems = ncols;
    if (do_givens && 3 * m + 1 > elems) elems = 3 * m + 1;
    size_t smem = (size_t)elems * sizeof(T);
    // Occupancy is computed for the largest request this kernel sees.
    const size_t smem_max = (size_t)(3 * MPK_MAX_STEPS + 8) * sizeof(T);
    int g = grid_for(kern, smem_max, n);
    kern<<<g, kBlock, smem, s>>>(n, V, ld, ncols, coef, w, wout, (T *)ws.partials, ws.counters, (T *)ws.sums, H,
                                 ctl, p, do_givens, done);
    return check_launch("k_update_norm");
}

template <typename T>
int launch_residual(const mpk_matrix *A, const T *b, const T *x, T *r, T *sums, float *rlow, float *sums_low,
                    Ws ws, cudaStream_t s) {
    return with_op<T>(A, [&](auto op) -> int {
        using Op = decltype(op);
        if (rlow) {
            if constexpr (sizeof(T) == 8) {
                auto kern = k_residual<T, Op, true>;
                int g = grid_for(kern, 0, op.n);
                kern<<<g, kBlock, 0, s>>>(op, b, x, r, rlow, (T *)ws.partials, ws.partials_low, ws.counters, sums,
                                          sums_low);
            } else {
                return fail(MPK_EARG, "low-precision residual copy needs an fp64 operator");
            }
        } else {
            auto kern = k_residual<T, Op, false>;
            int g = grid_for(kern, 0, op.n);
            kern<<<g, kBlock, 0, s>>>(op, b, x, r, nullptr, (T *)ws.partials, nullptr, ws.counters, sums, nullptr);
        }
        return check_launch("k_residual");
    });
}

// ---------------------------------------------------------------------------
// preconditioner application
// ---------------------------------------------------------------------------
template <typename T>
int apply_precond_t(const mpk_precond *M, const T *v, T *out, const int32_t *done, cudaStream_t s) {
    const int64_t n = M->n;
    if (M->kind == MPK_PC_NONE) {
        if (out != v) cudaMemcpyAsync(out, v, sizeof(T) * n, cudaMemcpyDeviceToDevice, s);
        return MPK_OK;
    }
    if (M->kind == MPK_PC_JACOBI) {
        const int k = M->block;
        const int64_t nb = (n + k - 1) / k;
        int g = (int)((nb + kBlock - 1) / kBlock);
        if (g > max_blocks()) g = max_blocks();
        if (g < 1) g = 1;
        if (k <= 8)
            k_jacobi<T, 8><<<g, kBlock, 0, s>>>(n, k, (const T *)M->lu, M->piv, v, out, done);
        else if (k <= 64)
            k_jacobi<T, 64><<<g, kBlock, 0, s>>>(n, k, (const T *)M->lu, M->piv, v, out, done);
        else
            return fail(MPK_EUNSUPPORTED, "block Jacobi block size > 64 not supported on device");
        return check_launch("k_jacobi");
    }
    if (M->kind == MPK_PC_POLY) {
        T *w1 = (T *)M->work, *w2 = w1 + n, *t = w2 + n;
        const T *work = v;
        int rc = MPK_OK;
        int i = 0;
        const int d = M->degree;
        bool first = true;
        while (i < d && rc == MPK_OK) {
            const double re = M->roots_re[i], im = M->roots_im[i];
            T *wnext = (work == w1) ? w2 : w1;
            if (im == 0.0) {   // preconditioners.py:293-297
                const double inv = 1.0 / re;
                const bool last = (i + 1 >= d);
                rc = with_op<T>(M->poly_A, [&](auto op) -> int {
                    using Op = decltype(op);
                    auto kern = k_poly_real<T, Op>;
                    int g = grid_for(kern, 0, op.n);
                    kern<<<g, kBlock, 0, s>>>(op, work, last ? nullptr : wnext, out, (T)inv, first ? 1 : 0, done);
                    return check_launch("k_poly_real");
                });
                i += 1;
            } else {           // preconditioners.py:298-304
                volatile double tr = 2.0 * re;
                volatile double rr = re * re;
                volatile double ii = im * im;
                const double m2 = rr + ii;
                const bool last = (i + 2 >= d);
                rc = with_op<T>(M->poly_A, [&](auto op) -> int {
                    using Op = decltype(op);
                    auto k1 = k_poly_pair1<T, Op>;
                    int g = grid_for(k1, 0, op.n);
                    k1<<<g, kBlock, 0, s>>>(op, work, t, out, (T)tr, (T)m2, first ? 1 : 0, done);
                    int rc1 = check_launch("k_poly_pair1");
                    if (rc1 || last) return rc1;
                    auto k2 = k_poly_pair2<T, Op>;
                    k2<<<g, kBlock, 0, s>>>(op, work, t, wnext, (T)tr, (T)m2, done);
                    return check_launch("k_poly_pair2");
                });
                i += 2;
            }
            first = false;
            work = wnext;
        }
        return rc;
    }
    return fail(MPK_EARG, "unknown preconditioner kind");
}

// M applied to a vector of the solver dtype T; a lower-precision M is
// wrapped cast-down / apply / cast-up (CastApplyPreconditioner,
// multiprecision.py:306-308).  Scratch for the cast lives after the poly work.
template <typename T>
int apply_precond(const mpk_precond *M, const T *v, T *out, const int32_t *done, cudaStream_t s) {
    const bool same = (M->dtype == MPK_F64) == (sizeof(T) == 8);
    if (same) return apply_precond_t<T>(M, v, out, done, s);
    if (M->dtype != MPK_F32 || sizeof(T) != 8) return fail(MPK_EARG, "preconditioner precision above solver precision");
    const int64_t n = M->n;
    float *lo_in = (float *)M->work + 3 * n, *lo_out = lo_in + n;
    int g = grid_for(k_convert_gated<double, float>, 0, n);
    k_convert_gated<double, float><<<g, kBlock, 0, s>>>(n, (const double *)v, lo_in, done);
    int rc = check_launch("k_convert_gated");
    if (rc) return rc;
    rc = apply_precond_t<float>(M, lo_in, lo_out, done, s);
    if (rc) return rc;
    k_convert_gated<float, double><<<g, kBlock, 0, s>>>(n, lo_out, (double *)out, done);
    return check_launch("k_convert_gated");
}

// ---------------------------------------------------------------------------
// one GMRES cycle
// ---------------------------------------------------------------------------
int64_t comm_part_core(int32_t dtype) { return 3LL * kFSlots * kXStride * (dtype == MPK_F64 ? 8 : 4); }

// the per-restart collectives' view of a communicator (comm.cuh); `dtype` =
// the precision set the buffers belong to
int comm_view(const mpk_comm *c, int32_t dtype, CommView &v) {
    memset(&v, 0, sizeof(v));
    if (!c || c->nranks < 1 || c->nranks > kMaxRanks || c->rank < 0 || c->rank >= c->nranks || !c->epoch)
        return fail(MPK_EARG, "inconsistent mpk_comm");
    v.rank = c->rank;
    v.nranks = c->nranks;
    v.row0 = c->row0;
    v.epoch = (unsigned long long *)c->epoch;
    const int64_t core = comm_part_core(dtype);
    for (int q = 0; q < c->nranks; ++q) {
        if (!c->part[q] || !c->xbar[q] || !c->xg[q]) return fail(MPK_EARG, "null peer pointer");
        v.xg[q] = (char *)c->xg[q];
        v.xbar[q] = (unsigned long long *)c->xbar[q];
        v.scal[q] = (char *)c->part[q] + core;
        v.mir_lo[q] = c->mir_lo[q];
        v.mir_hi[q] = c->mir_hi[q];
    }
    return MPK_OK;
}

// CTAs of the persistent cycle: one per SM, at least 64 rows each
// (measured on C1, 64k rows: 148 CTAs 23.0 us/iteration, 64 CTAs 24.8,
// 16 CTAs 38.7 -- the barriers do not get cheaper with fewer arrivals).
// MPK_FUSED_ROWS_PER_CTA / MPK_FUSED_CTAS override.
int fused_grid(int sms, int64_t n) {
    static int force = -1, min_rows = -1;
    if (force < 0) {
        const char *e = getenv("MPK_FUSED_CTAS");
        force = e ? atoi(e) : 0;
        const char *r = getenv("MPK_FUSED_ROWS_PER_CTA");
        min_rows = r ? atoi(r) : 64;
        if (min_rows < 64) min_rows = 64;
    }
    if (force > 0) return force < sms ? force : sms;
    int64_t g = n / min_rows;
    if (g < 1) g = 1;
    return g < sms ? (int)g : sms;
}

// Row-partitioned cycles: the rank's view of the communicator into the
// kernel arguments (w'' / the candidate live in the rank's global-length x
// buffer); the CTA count is the communicator's (all ranks must agree).
template <typename T> int fill_comm(FusedArgs<T> &fa, const mpk_cycle_desc *d, int &grid) {
    memset(&fa.cm, 0, sizeof(fa.cm));
    fa.cm.nranks = 1;
    if (d->nranks > 1) {
        const mpk_comm *c = d->comm;
        if (!c || c->nranks != d->nranks || c->nranks > kMaxRanks || c->rank < 0 || c->rank >= c->nranks)
            return fail(MPK_EARG, "multi-rank cycle needs a consistent mpk_comm");
        fa.cm.rank = c->rank;
        fa.cm.nranks = c->nranks;
        fa.cm.row0 = c->row0;
        fa.cm.epoch = (unsigned long long *)c->epoch;
        for (int q = 0; q < c->nranks; ++q) {
            fa.cm.part[q] = (T *)c->part[q];
            fa.cm.xbar[q] = (unsigned long long *)c->xbar[q];
            fa.cm.xg[q] = (T *)c->xg[q];
            fa.cm.mir_lo[q] = c->mir_lo[q];
            fa.cm.mir_hi[q] = c->mir_hi[q];
            if (!fa.cm.part[q] || !fa.cm.xbar[q] || !fa.cm.xg[q]) return fail(MPK_EARG, "null peer pointer");
        }
        if (c->row0 % 64 != 0 || ((uintptr_t)c->xg[c->rank] % 16) != 0)
            return fail(MPK_EARG, "rank row blocks must start on 64-row boundaries");
        fa.wpp = (T *)c->xg[c->rank] + c->row0;   // w'' lives in the rank's global-length vector
        if (c->ctas > 0 && c->ctas < grid) grid = c->ctas;
    }
    return MPK_OK;
}

// k_cycle_reg launch; TV = __half stores the basis in binary16 (desc flag
// bit 5: fp32 cycles on one GPU, m <= 51), scaled by vs = 2^round(log2
// sqrt(n)) so normalised basis entries sit in binary16's normal range.
// L2 persistence for the cycle's work vectors (w, w', w''), re-read within
// every Arnoldi step while the basis streams through L2: a persisting
// set-aside of ~32 MB (set once, only if the process has none; MPK_L2_PERSIST=0
// disables) and a per-launch access-policy window over the first vectors
// (hitRatio 1).  Measured with tools/l2_persist_probe.py: C2 1.02-1.03x,
// C4 1.01-1.02x; larger set-asides cost the basis its L2 reuse.
// mpk_l2_release() returns the persisting lines to normal after a solve.
size_t l2_persist_bytes() {
    static int state = -1;   // -1 unknown, else set-aside bytes (0: off)
    static size_t aside = 0;
    if (state < 0) {
        const char *e = getenv("MPK_L2_PERSIST");
        const bool on = !(e && atoi(e) == 0);
        size_t cur = 0;
        if (on && cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) == cudaSuccess) {
            if (cur == 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)32 << 20) == cudaSuccess)
                cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            aside = cur;
        }
        cudaGetLastError();   // a refused limit is not an error of the solve
        state = aside > 0 ? 1 : 0;
    }
    return aside;
}

// Resident CTAs per SM of a persistent cycle kernel at `smem` bytes of
// dynamic shared memory, cached per (kernel, smem): the occupancy query costs
// tens of microseconds of host time, and it used to run before every cycle
// launch (on the GPU-idle path between refinements).
int coop_per_sm(const void *kern, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void *, size_t>, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(kern, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFB, smem);
    cache[key] = per_sm;
    return per_sm;
}

// Cooperative launch of a persistent cycle kernel, with the L2 window over
// [win, win + win_bytes) when persistence is available.
cudaError_t launch_cycle_coop(const void *kern, int grid, size_t smem, cudaStream_t s, void **args, const void *win,
                              size_t win_bytes) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kFB);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    int na = 1;
    const size_t aside = l2_persist_bytes();
    if (aside > 0 && win && win_bytes > 0) {
        at[1].id = cudaLaunchAttributeAccessPolicyWindow;
        at[1].val.accessPolicyWindow.base_ptr = const_cast<void *>(win);
        at[1].val.accessPolicyWindow.num_bytes = win_bytes < aside ? win_bytes : aside;
        at[1].val.accessPolicyWindow.hitRatio = 1.0f;
        at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        na = 2;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelExC(&cfg, kern, args);
}

template <typename T, class Op, typename TV = T>
int launch_fused_reg(const Op &op, const mpk_cycle_desc *d, int cap, double tf, double u, cudaStream_t s) {
    const int m = d->m;
    T *w = (T *)d->work;
    Ws ws = carve(d->ws);
    // layout of k_cycle_reg: small m keeps R (m+1 x m) in shared memory
    const bool big = m + 1 > kRegMaxCols;
    const bool multi = d->nranks > 1;
    constexpr bool half = !std::is_same<T, TV>::value;
    if (multi && big) return fail(MPK_EUNSUPPORTED, "row-partitioned cycles support m <= 51");
    if (half && (multi || big)) return fail(MPK_EUNSUPPORTED, "binary16 basis: one GPU, m <= 51");
    const bool poly = d->M && d->M->kind == MPK_PC_POLY;
    if (poly && (half || multi || big)) return fail(MPK_EUNSUPPORTED, "polynomial cycle: one GPU, m <= 51");
    void (*kern)(Op, FusedArgs<T>);
    if constexpr (half) kern = k_cycle_reg<T, Op, false, false, TV>;
    else kern = poly ? k_cycle_reg<T, Op, false, false, T, true>
                     : multi ? k_cycle_reg<T, Op, false, true>
                             : (big ? k_cycle_reg<T, Op, true, false> : k_cycle_reg<T, Op, false, false>);
    const size_t nslot = big ? (size_t)m + 2 : (size_t)kFSlots;
    // (banded CSR: staging x in a shared-memory window for phase A's SpMV,
    // as k_spmv_win does, measured slower inside the cycle -- C5 IR 0.774 vs
    // 0.690 s, profiles/r02_C5_window_ab.txt -- so the cycle gathers via L1)
    const size_t smem = sizeof(T) * ((big ? 0 : (size_t)(m + 1) * m) + 2 * m + (m + 1) + 2 * nslot + kFW * kFSlots +
                                     (big ? nslot : 0) + kFW * kCsrWarpBuf);
    static size_t attr_set[4] = {0, 0, 0, 0};   // per kernel (TV is a template parameter)
    const int vi = poly ? 3 : multi ? 2 : (big ? 1 : 0);
    if (smem > attr_set[vi]) {
        cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) {
            g_err = std::string("k_cycle_reg smem attribute: ") + cudaGetErrorString(ea);
            return MPK_ELAUNCH;
        }
        attr_set[vi] = smem;
    }
    if (coop_per_sm((const void *)kern, smem) < 1) return fail(MPK_ELAUNCH, "register cycle kernel does not fit on an SM");
    int grid = sm_count_cached();
    if (grid > kFMaxCtas) grid = kFMaxCtas;
    if (d->nranks <= 1) grid = fused_grid(grid, d->n);   // ranks must agree on the CTA count (partial columns)
    FusedArgs<T> fa;
    fa.n = d->n;
    fa.ld = d->ld;
    fa.m = m;
    fa.cap = cap;
    fa.V = (T *)d->V;
    fa.r0 = (const T *)d->r0;
    fa.rnorm2 = (const T *)d->rnorm2;
    fa.x0 = (const T *)d->x0;
    fa.x_out = (T *)d->x_out;
    fa.w = w;
    fa.wp = w + d->ld;
    fa.wpp = w + 2 * d->ld;
    fa.part = (T *)ws.partials;
    fa.bar = ws.counters + 8;
    fa.H = hess_view<T>(d->hess, m);
    fa.ctl = d->ctl;
    fa.tf = tf;
    fa.exit_tol = d->exit_tol;
    fa.norm_scale = d->norm_scale;
    fa.u = u;
    fa.final_col = (d->flags & 2) ? 1 : 0;
    fa.prof = (d->flags & 8) ? 1 : 0;
    fa.diag = nullptr;
    fa.z = w + 3 * d->ld;
    if (d->M && d->M->kind == MPK_PC_POLY) {
        // units of the product form with the multi-kernel path's host
        // arithmetic (apply_precond_t): inv = 1/re; tr = 2 re, m2 = re^2 + im^2
        const mpk_precond *M = d->M;
        int nu = 0;
        for (int i = 0; i < M->degree;) {
            if (nu >= kMaxPolyUnits) return fail(MPK_EUNSUPPORTED, "polynomial degree too high for the fused cycle");
            const double re = M->roots_re[i], im = M->roots_im[i];
            if (im == 0.0) {
                fa.poly[nu].pair = 0;
                fa.poly[nu].a = (T)(1.0 / re);
                fa.poly[nu].b = T(0);
                i += 1;
            } else {
                volatile double tr = 2.0 * re;
                volatile double rr = re * re;
                volatile double ii = im * im;
                const double m2 = rr + ii;
                fa.poly[nu].pair = 1;
                fa.poly[nu].a = (T)tr;
                fa.poly[nu].b = (T)m2;
                i += 2;
            }
            ++nu;
        }
        fa.npoly = nu;
        const int64_t pn = M->n;
        fa.pw0 = (T *)M->work;
        fa.pw1 = fa.pw0 + pn;
        fa.pt = fa.pw1 + pn;
        fa.pacc = w + 3 * d->ld;
    }
    if constexpr (half) {
        const double e = std::nearbyint(0.5 * std::log2((double)(d->n > 1 ? d->n : 1)));
        fa.vs = (T)std::ldexp(1.0, (int)e);
        fa.vsi = (T)std::ldexp(1.0, -(int)e);
    }
    if (d->M && d->M->kind == MPK_PC_JACOBI && d->M->block == 1 && d->M->dtype == d->dtype)
        fa.diag = (const T *)d->M->lu;
    if (int rc = fill_comm<T>(fa, d, grid)) return rc;
    if constexpr (Op::kStencil) {
        // 3-D stencils reach +-nx^2 rows, about a CTA's slab at C4: one more
        // grid barrier per step lets the SpMV read v_k's halo from the stored
        // column instead of dividing w'' by beta again (MPK_VK_SYNC=0/1 overrides)
        static int force = -2;
        if (force == -2) {
            const char *e = getenv("MPK_VK_SYNC");
            force = e ? atoi(e) : -1;
        }
        const int64_t reach = op.k.preset == MPK_LAPLACE3D ? (int64_t)op.k.nx * op.k.nx : (int64_t)op.k.nx + 1;
        const int64_t rpc = ((d->n + grid - 1) / grid + 63) / 64 * 64;
        fa.vk_sync = (!multi && !poly && (force >= 0 ? force : (2 * reach > rpc && rpc >= 16384))) ? 1 : 0;
    }
    Op opc = op;
    void *args[] = {(void *)&opc, (void *)&fa};
    ProfScope ps(7, 0.0, s);
    // one GPU: the work vectors w, w', w'' in the L2 window (row-partitioned
    // cycles keep plain cooperative launches: their buffers are peer-mapped)
    cudaError_t e = launch_cycle_coop((const void *)kern, grid, smem, s, args, multi ? nullptr : (const void *)w,
                                      3 * (size_t)d->ld * sizeof(T));
    if (e != cudaSuccess) {
        g_err = std::string("k_cycle_reg: ") + cudaGetErrorString(e);
        return MPK_ELAUNCH;
    }
    g_last_cycle = half ? (std::is_same<TV, __half>::value ? "k_cycle_reg/half" : "k_cycle_reg/bf16")
                        : poly ? "k_cycle_reg/poly" : multi ? "k_cycle_reg/multi" : (big ? "k_cycle_reg/big" : "k_cycle_reg");
    return check_launch("k_cycle_reg");
}

// Lagged one-reduction CGS2 (desc flag bit 4, SolverConfig.orthogonalization
// = "dcgs2"): identity preconditioner, m <= 51, one GPU.
// TV: basis storage (T, or a 16-bit basis on one GPU, flags 32 / 64).
template <typename T, class Op, typename TV = T>
int launch_dcgs2(const Op &op, const mpk_cycle_desc *d, int cap, double tf, double u, cudaStream_t s) {
    const int m = d->m;
    T *w = (T *)d->work;
    Ws ws = carve(d->ws);
    constexpr bool half = sizeof(TV) != sizeof(T);
    auto kern = k_cycle_dcgs2<T, Op, false, TV>;
    if constexpr (!half) {
        if (d->nranks > 1) kern = k_cycle_dcgs2<T, Op, true, TV>;
    }
    const size_t smem = sizeof(T) * (2 * (size_t)(m + 1) * m + 2 * m + (m + 1) + 5 * 64 + kFW * kFSlots +
                                     kFW * kCsrWarpBuf);
    static size_t attr_set[2] = {0, 0};
    const int mi = d->nranks > 1 ? 1 : 0;
    if (smem > attr_set[mi]) {
        cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) {
            g_err = std::string("k_cycle_dcgs2 smem attribute: ") + cudaGetErrorString(ea);
            return MPK_ELAUNCH;
        }
        attr_set[mi] = smem;
    }
    if (coop_per_sm((const void *)kern, smem) < 1) return fail(MPK_ELAUNCH, "dcgs2 cycle kernel does not fit on an SM");
    int grid = sm_count_cached();
    if (grid > 160) grid = 160;   // cross_reduce fast path
    if (d->nranks <= 1) grid = fused_grid(grid, d->n);
    FusedArgs<T> fa;
    memset(&fa, 0, sizeof(fa));
    fa.n = d->n;
    fa.ld = d->ld;
    fa.m = m;
    fa.cap = cap;
    fa.V = (T *)d->V;
    fa.r0 = (const T *)d->r0;
    fa.rnorm2 = (const T *)d->rnorm2;
    fa.x0 = (const T *)d->x0;
    fa.x_out = (T *)d->x_out;
    fa.w = w;
    fa.wp = w + d->ld;
    fa.wpp = w + 2 * d->ld;
    fa.part = (T *)ws.partials;
    fa.bar = ws.counters + 8;
    fa.H = hess_view<T>(d->hess, m);
    fa.ctl = d->ctl;
    fa.tf = tf;
    fa.exit_tol = d->exit_tol;
    fa.norm_scale = d->norm_scale;
    fa.u = u;
    fa.diag = nullptr;
    fa.z = w + 3 * d->ld;
    fa.vs = fa.vsi = T(1);
    if constexpr (half) {
        // the same power-of-two scale as k_cycle_reg's 16-bit basis
        const double e = std::nearbyint(0.5 * std::log2((double)(d->n > 1 ? d->n : 1)));
        fa.vs = (T)std::ldexp(1.0, (int)e);
        fa.vsi = (T)std::ldexp(1.0, -(int)e);
    }
    if (d->M && d->M->kind == MPK_PC_JACOBI && d->M->block == 1 && d->M->dtype == d->dtype)
        fa.diag = (const T *)d->M->lu;
    if (int rc = fill_comm<T>(fa, d, grid)) return rc;
    Op opc = op;
    void *args[] = {(void *)&opc, (void *)&fa};
    ProfScope ps(7, 0.0, s);
    cudaError_t e = launch_cycle_coop((const void *)kern, grid, smem, s, args,
                                      d->nranks > 1 ? nullptr : (const void *)w, 3 * (size_t)d->ld * sizeof(T));
    if (e != cudaSuccess) {
        g_err = std::string("k_cycle_dcgs2: ") + cudaGetErrorString(e);
        return MPK_ELAUNCH;
    }
    g_last_cycle = half ? (std::is_same<TV, __half>::value ? "k_cycle_dcgs2/half" : "k_cycle_dcgs2/bf16")
                        : d->nranks > 1 ? "k_cycle_dcgs2/multi" : "k_cycle_dcgs2";
    return check_launch("k_cycle_dcgs2");
}

template <typename T> int run_cycle(const mpk_cycle_desc *d, cudaStream_t s) {
    const int64_t n = d->n, ld = d->ld;
    const int m = d->m;
    if (m < 1 || m > MPK_MAX_STEPS - 1) return fail(MPK_EARG, "restart length out of range");
    const int cap = d->steps_cap < 1 ? 1 : (d->steps_cap > m ? m : d->steps_cap);
    const int sv = sizeof(T);
    T *V = (T *)d->V;
    T *w = (T *)d->work, *wp = w + ld, *wpp = wp + ld, *z = wpp + ld;
    Ws ws = carve(d->ws);
    T *sums = (T *)ws.sums;
    Hess<T> H = hess_view<T>(d->hess, m);
    mpk_cycle_ctl *ctl = d->ctl;
    const int32_t *done = &ctl->done;
    const bool precond = d->M != nullptr && d->M->kind != MPK_PC_NONE;
    const double u = (sizeof(T) == 8) ? std::ldexp(1.0, -53) : std::ldexp(1.0, -24);
    const double tf = (d->rule == MPK_RULE_U) ? u : (double)n * u;   // kernels.py:122
    int rc;

    if (d->nranks > 1) {
        // identity, or block Jacobi(1) whose `lu` is the GLOBAL diagonal
        // offset to the rank's first row (halo rows read their own a_ii)
        const bool jac1 = precond && d->M->kind == MPK_PC_JACOBI && d->M->block == 1 && d->M->n == n &&
                          d->M->dtype == d->dtype && (uintptr_t)d->M->lu % 16 == 0;
        if ((precond && !jac1) || m + 1 > kRegMaxCols || (uintptr_t)d->x_out % 16 || (uintptr_t)d->V % 16 ||
            (uintptr_t)d->work % 16 || (uintptr_t)d->r0 % 16)
            return fail(MPK_EUNSUPPORTED, "row-partitioned cycle: identity or Jacobi(1) preconditioner, m <= 51, "
                                          "16-byte aligned buffers");
        if ((d->flags & 16) && !precond)   // lagged one-reduction CGS2, row-partitioned instantiation
            return with_op<T>(d->A, [&](auto op) -> int { return launch_dcgs2<T, decltype(op)>(op, d, cap, tf, u, s); });
        return with_op<T>(d->A, [&](auto op) -> int {
            return launch_fused_reg<T, decltype(op)>(op, d, cap, tf, u, s);
        });
    }
    // block Jacobi with 1x1 blocks is a diagonal scaling: the persistent
    // register kernel applies it inside its SpMV input and correction
    const bool diag1 = precond && d->M->kind == MPK_PC_JACOBI && d->M->block == 1 && d->M->n == n &&
                       d->M->dtype == d->dtype;
    if (d->flags & (32 | 64)) {
        // 16-bit basis storage (SolverConfig.basis_precision = "binary16" /
        // "bfloat16")
        if constexpr (sizeof(T) == 4) {
            const bool ok = (!precond || diag1) && !(d->flags & 4) && d->nranks <= 1 &&
                            m + 1 <= kRegMaxCols && (uintptr_t)d->x_out % 16 == 0 && (uintptr_t)d->V % 16 == 0 &&
                            (uintptr_t)d->work % 16 == 0 && (uintptr_t)d->r0 % 16 == 0 &&
                            (d->flags & (32 | 64)) != (32 | 64);
            if (!ok)
                return fail(MPK_EUNSUPPORTED, "16-bit basis: one GPU, m <= 51, identity or Jacobi(1)");
            if (d->flags & 16)   // lagged one-reduction CGS2 over the 16-bit basis
                return with_op<T>(d->A, [&](auto op) -> int {
                    if (d->flags & 64) return launch_dcgs2<T, decltype(op), __nv_bfloat16>(op, d, cap, tf, u, s);
                    return launch_dcgs2<T, decltype(op), __half>(op, d, cap, tf, u, s);
                });
            return with_op<T>(d->A, [&](auto op) -> int {
                if (d->flags & 64) return launch_fused_reg<T, decltype(op), __nv_bfloat16>(op, d, cap, tf, u, s);
                return launch_fused_reg<T, decltype(op), __half>(op, d, cap, tf, u, s);
            });
        } else {
            return fail(MPK_EUNSUPPORTED, "16-bit basis storage needs binary32 cycles");
        }
    }
    if ((d->flags & 16) && (!precond || (diag1 && d->nranks <= 1)) && m + 1 <= kRegMaxCols &&
        (uintptr_t)d->x_out % 16 == 0 &&
        (uintptr_t)d->V % 16 == 0 && (uintptr_t)d->work % 16 == 0 && (uintptr_t)d->r0 % 16 == 0) {
        return with_op<T>(d->A, [&](auto op) -> int { return launch_dcgs2<T, decltype(op)>(op, d, cap, tf, u, s); });
    }
    // identity preconditioner, any m: the persistent register kernel (column
    // blocks beyond 51 columns)
    if (!precond && !(d->flags & 4) && (uintptr_t)d->x_out % 16 == 0 &&
        (uintptr_t)d->V % 16 == 0 && (uintptr_t)d->work % 16 == 0 && (uintptr_t)d->r0 % 16 == 0) {
        return with_op<T>(d->A, [&](auto op) -> int {
            return launch_fused_reg<T, decltype(op)>(op, d, cap, tf, u, s);
        });
    }
    // GMRES polynomial on the cycle's own operator: applied inside the
    // persistent register kernel (one grid barrier per SpMV)
    const bool poly_fused = precond && d->M->kind == MPK_PC_POLY && d->M->dtype == d->dtype && d->M->n == n &&
                            d->nranks <= 1 && m + 1 <= kRegMaxCols && !(d->flags & 4) && d->M->work &&
                            d->M->poly_A && same_operator(d->M->poly_A, d->A);
    if (poly_fused && (uintptr_t)d->x_out % 16 == 0 && (uintptr_t)d->V % 16 == 0 &&
        (uintptr_t)d->work % 16 == 0 && (uintptr_t)d->r0 % 16 == 0 && (uintptr_t)d->M->work % 16 == 0) {
        return with_op<T>(d->A, [&](auto op) -> int {
            return launch_fused_reg<T, decltype(op)>(op, d, cap, tf, u, s);
        });
    }
    if (diag1 && m + 1 <= kRegMaxCols && !(d->flags & 4) &&
        (uintptr_t)d->x_out % 16 == 0 && (uintptr_t)d->V % 16 == 0 && (uintptr_t)d->work % 16 == 0 &&
        (uintptr_t)d->r0 % 16 == 0 && (uintptr_t)d->M->lu % 16 == 0) {
        return with_op<T>(d->A, [&](auto op) -> int {
            return launch_fused_reg<T, decltype(op)>(op, d, cap, tf, u, s);
        });
    }
    g_last_cycle = "multi-kernel";
    k_cycle_begin<T><<<1, 32, 0, s>>>((const T *)d->rnorm2, sums, H, ctl, d->norm_scale);
    if ((rc = check_launch("k_cycle_begin"))) return rc;

    for (int k = 0; k < cap; ++k) {
        const int ncols = k + 1;
        const T *src = (k == 0) ? (const T *)d->r0 : wpp;
        const T *divp = (k == 0) ? sums + S_GAMMA : sums + S_BETA;
        T *vcol = V + (int64_t)k * ld;
        const double vbytes = (double)sv * n * ncols;
        if (!precond) {
            ProfScope ps(0, spmv_bytes(d->A, sv) + 2.0 * sv * n + vbytes, s);
            if (ncols <= kMaxCols) {
                rc = with_op<T>(d->A, [&](auto op) -> int {
                    return launch_p1<T, decltype(op), true>(op, src, divp, vcol, V, ld, ncols, w, ws, sums + S_C1,
                                                           sums + S_WN2, done, s);
                });
            } else {
                rc = with_op<T>(d->A, [&](auto op) -> int {
                    return launch_p1<T, decltype(op), true>(op, src, divp, vcol, V, ld, 0, w, ws, sums + S_TMP,
                                                           sums + S_WN2, done, s);
                });
                if (!rc) rc = launch_multidot<T>(n, V, ld, ncols, w, ws, sums + S_C1, done, s);
            }
        } else {
            {
                ProfScope ps(3, 2.0 * sv * n, s);
                int g = grid_for(k_normalize<T>, 0, n);
                k_normalize<T><<<g, kBlock, 0, s>>>(n, src, divp, vcol, done);
                if ((rc = check_launch("k_normalize"))) return rc;
            }
            {
                ProfScope ps(4, 0.0, s);
                if ((rc = apply_precond<T>(d->M, vcol, z, done, s))) return rc;
            }
            ProfScope ps(0, spmv_bytes(d->A, sv) + sv * n + vbytes, s);
            if (ncols <= kMaxCols) {
                rc = with_op<T>(d->A, [&](auto op) -> int {
                    return launch_p1<T, decltype(op), false>(op, z, divp, vcol, V, ld, ncols, w, ws, sums + S_C1,
                                                            sums + S_WN2, done, s);
                });
            } else {
                rc = with_op<T>(d->A, [&](auto op) -> int {
                    return launch_p1<T, decltype(op), false>(op, z, divp, vcol, V, ld, 0, w, ws, sums + S_TMP,
                                                            sums + S_WN2, done, s);
                });
                if (!rc) rc = launch_multidot<T>(n, V, ld, ncols, w, ws, sums + S_C1, done, s);
            }
        }
        if (rc) return rc;
        {
            ProfScope ps(1, vbytes + 2.0 * sv * n, s);
            if (ncols <= kMaxCols) {
                rc = launch_p2<T>(n, V, ld, ncols, sums + S_C1, w, wp, ws, sums + S_C2, done, s);
            } else {
                rc = launch_p3<T>(n, V, ld, ncols, sums + S_C1, w, wp, ws, H, ctl, StepParams{k, cap, tf, d->exit_tol, 1},
                                  0, done, s);
                if (!rc) rc = launch_multidot<T>(n, V, ld, ncols, wp, ws, sums + S_C2, done, s);
            }
            if (rc) return rc;
        }
        {
            ProfScope ps(2, vbytes + 2.0 * sv * n, s);
            rc = launch_p3<T>(n, V, ld, ncols, sums + S_C2, wp, wpp, ws, H, ctl, StepParams{k, cap, tf, d->exit_tol, 1}, 1,
                              done, s);
            if (rc) return rc;
        }
    }
    if (d->flags & 2) {
        int gf = grid_for(k_final_column<T>, 0, n);
        k_final_column<T><<<gf, kBlock, 0, s>>>(n, wpp, sums + S_BETA, V, ld, ctl);
        if ((rc = check_launch("k_final_column"))) return rc;
    }
    // epilogue: d = R \ g ; x_out = x0 + M(V_k d)
    k_lsq_solve<T><<<1, 32, (size_t)(m + 1) * sizeof(T), s>>>(H, ctl, u, 0);
    if ((rc = check_launch("k_lsq_solve"))) return rc;
    ProfScope ps(5, (double)sv * n * (cap + 2), s);
    const size_t smem = (size_t)(m + 1) * sizeof(T);
    int g = grid_for(k_correct<T>, smem, n);
    if (!precond) {
        k_correct<T><<<g, kBlock, smem, s>>>(n, V, ld, H.d, (const T *)d->x0, (T *)d->x_out, ctl, 0);
        return check_launch("k_correct");
    }
    k_correct<T><<<g, kBlock, smem, s>>>(n, V, ld, H.d, nullptr, w, ctl, 1);
    if ((rc = check_launch("k_correct"))) return rc;
    // M(y): gated on the triangular-breakdown flag through a scratch int is
    // unnecessary — a failed solve leaves x_out untouched below.
    if ((rc = apply_precond<T>(d->M, w, z, nullptr, s))) return rc;
    int g2 = grid_for(k_add_gated<T>, 0, n);
    k_add_gated<T><<<g2, kBlock, 0, s>>>(n, (const T *)d->x0, z, (T *)d->x_out, ctl);
    return check_launch("k_add_gated");
}

template <typename T>
int cgs2_append_t(int64_t n, int64_t ld, int count, T *V, const T *w, int rule, T *coeffs, T *out, int32_t *app,
                  T *tmp, Ws ws, cudaStream_t s) {
    T *sums = (T *)ws.sums;
    T *wp = tmp, *wpp = tmp + n;
    int rc;
    const double u = (sizeof(T) == 8) ? std::ldexp(1.0, -53) : std::ldexp(1.0, -24);
    const double tf = (rule == MPK_RULE_U) ? u : (double)n * u;
    // ||w||^2 and c1 (multidot's extra slot carries w.w)
    {
        auto kern = k_dot<T>;
        int g = grid_for(kern, 0, n);
        kern<<<g, kBlock, 0, s>>>(n, w, w, (T *)ws.partials, ws.counters, sums + S_WN2, 0);
        if ((rc = check_launch("k_dot"))) return rc;
    }
    if ((rc = launch_multidot<T>(n, V, ld, count, w, ws, sums + S_C1, nullptr, s))) return rc;
    Hess<T> H{};
    if (count <= kMaxCols) {
        if ((rc = launch_p2<T>(n, V, ld, count, sums + S_C1, w, wp, ws, sums + S_C2, nullptr, s))) return rc;
    } else {
        if ((rc = launch_p3<T>(n, V, ld, count, sums + S_C1, w, wp, ws, H, nullptr, StepParams{0, 1, tf, 0.0, 0}, 0,
                               nullptr, s)))
            return rc;
        if ((rc = launch_multidot<T>(n, V, ld, count, wp, ws, sums + S_C2, nullptr, s))) return rc;
    }
    if ((rc = launch_p3<T>(n, V, ld, count, sums + S_C2, wp, wpp, ws, H, nullptr, StepParams{0, 1, tf, 0.0, 0}, 0,
                           nullptr, s)))
        return rc;
    int g = grid_for(k_cgs2_finish<T>, 0, n);
    k_cgs2_finish<T><<<g, kBlock, 0, s>>>(n, sums, count, tf, wpp, V + (int64_t)count * ld, coeffs, out, app);
    return check_launch("k_cgs2_finish");
}

}  // namespace

// ===========================================================================
// extern "C" ABI
// ===========================================================================
extern "C" {

int mpk_abi_version(void) { return MPK_ABI_VERSION; }
const char *mpk_last_error(void) { return g_err.c_str(); }
int mpk_sm_count(void) { return sm_count_cached(); }

int mpk_l2_release(void) {
    if (l2_persist_bytes() == 0) return MPK_OK;
    cudaError_t e = cudaCtxResetPersistingL2Cache();
    if (e != cudaSuccess) {
        g_err = std::string("cudaCtxResetPersistingL2Cache: ") + cudaGetErrorString(e);
        return MPK_ELAUNCH;
    }
    return MPK_OK;
}

int64_t mpk_reduce_ws_bytes(int64_t n, int32_t max_cols) {
    (void)n;
    (void)max_cols;
    return 256 + align_up(ws_partials_bytes(), 256) + align_up(ws_low_bytes(), 256) + (int64_t)S_TOTAL * 8 + 256;
}

int64_t mpk_cycle_hess_bytes(int32_t m, int32_t dtype) {
    const int64_t sv = dtype == MPK_F64 ? 8 : 4;
    return sv * (2 * (int64_t)(m + 1) * m + m + m + (m + 1) + m) + 64;
}

int mpk_spmv(const mpk_matrix *A, const void *x, void *y, void *stream) {
    if (!A || !x || !y) return fail(MPK_EARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    auto go = [&](auto tag) -> int {
        using T = decltype(tag);
        return with_op<T>(A, [&](auto op) -> int {
            using Op = decltype(op);
            if (op.n == 0) return MPK_OK;
            if constexpr (!Op::kStencil) {
                // row split chosen by row-length statistics (north_star (1)):
                // short rows thread per row, long banded rows warp-cooperative
                // with an x window, other long rows warp-cooperative
                if (A->nnz <= 8 * A->n) {
                    auto kr = k_spmv_rows<T>;
                    int g = grid_for(kr, 0, (op.n + 1) / 2);
                    kr<<<g, kBlock, 0, s>>>(op, (const T *)x, (T *)y);
                    return check_launch("k_spmv_rows");
                }
                const int64_t we = csr_window_elems(op, kSpmvChunk);
                if (we > 0) {
                    // banded rows: x window in shared memory; 16 entries per
                    // lane when rows are long (config 5: ~49 entries)
                    auto kw = k_spmv_win<T, 8>;   // gathers hit shared memory: 8 entries per lane suffice
                    const size_t smem = (size_t)we * sizeof(T);
                    // the window replaces L1 reuse: prefer shared memory so
                    // occupancy is not capped by the default carveout
                    static bool carve = false;
                    if (!carve) {
                        cudaFuncSetAttribute(k_spmv_win<T, 8>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             (int)cudaSharedmemCarveoutMaxShared);
                        carve = true;
                    }
                    int g = grid_for(kw, smem, (op.n + kSpmvChunk - 1) / kSpmvChunk * kBlock);
                    kw<<<g, kBlock, smem, s>>>(op, (const T *)x, (T *)y);
                    return check_launch("k_spmv_win");
                }
            }
            if constexpr (Op::kStencil) {
                // row groups with the preset fixed at compile time
                // (k_spmv_pre), one group per thread and trip: measured
                // against the generic k_spmv (profiles/r02_spmv_pre_ab.txt)
                // Laplace3D 200^3 55 -> 62% (fp64) and 55 -> 64% (fp32) of
                // the copy peak, the 2-D presets unchanged; two groups per
                // trip took 99 registers and fell to 37% in fp64
                constexpr int R = 16 / (int)sizeof(T);
                // StencilOp::group_ok() evaluated on the host side
                const bool groups = op.k.preset != MPK_STRETCHED2D && op.k.nx % R == 0 && op.k.row0 % R == 0;
                if (groups && ((uintptr_t)x % 16) == 0 && ((uintptr_t)y % 16) == 0) {
                    void (*kp)(StencilOp<T>, const T *, T *) = nullptr;
                    switch (op.k.preset) {
                        case MPK_LAPLACE3D: kp = k_spmv_pre<T, MPK_LAPLACE3D, 1>; break;
                        case MPK_LAPLACE2D: kp = k_spmv_pre<T, MPK_LAPLACE2D, 1>; break;
                        case MPK_UNIFLOW2D: kp = k_spmv_pre<T, MPK_UNIFLOW2D, 1>; break;
                        case MPK_BENTPIPE2D: kp = k_spmv_pre<T, MPK_BENTPIPE2D, 1>; break;
                        default: break;
                    }
                    if (kp) {
                        int g = grid_for(kp, 0, op.n / R);
                        kp<<<g, kBlock, 0, s>>>(op, (const T *)x, (T *)y);
                        return check_launch("k_spmv_pre");
                    }
                }
            }
            auto kern = k_spmv<T, Op>;
            int g = grid_for(kern, 0, op.n);
            kern<<<g, kBlock, 0, s>>>(op, (const T *)x, (T *)y);
            return check_launch("k_spmv");
        });
    };
    return A->dtype == MPK_F64 ? go(double{}) : go(float{});
}

int mpk_convert(int32_t sd, int32_t dd, int64_t n, const void *src, void *dst, void *stream) {
    if (n == 0) return MPK_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (sd == dd) {
        cudaMemcpyAsync(dst, src, n * (sd == MPK_F64 ? 8 : 4), cudaMemcpyDeviceToDevice, s);
        return check_launch("convert copy");
    }
    if (sd == MPK_F64) {
        int g = grid_for(k_convert<double, float>, 0, n);
        k_convert<double, float><<<g, kBlock, 0, s>>>(n, (const double *)src, (float *)dst);
    } else {
        int g = grid_for(k_convert<float, double>, 0, n);
        k_convert<float, double><<<g, kBlock, 0, s>>>(n, (const float *)src, (double *)dst);
    }
    return check_launch("k_convert");
}

int mpk_vdiv(int32_t dtype, int64_t n, const void *x, const void *d, void *out, void *stream) {
    if (n == 0) return MPK_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == MPK_F64) {
        int g = grid_for(k_normalize<double>, 0, n);
        k_normalize<double><<<g, kBlock, 0, s>>>(n, (const double *)x, (const double *)d, (double *)out, nullptr);
    } else {
        int g = grid_for(k_normalize<float>, 0, n);
        k_normalize<float><<<g, kBlock, 0, s>>>(n, (const float *)x, (const float *)d, (float *)out, nullptr);
    }
    return check_launch("k_normalize");
}

int mpk_dot(int32_t dtype, int64_t n, const void *x, const void *y, void *result, void *ws_, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Ws ws = carve(ws_);
    if (dtype == MPK_F64) {
        int g = grid_for(k_dot<double>, 0, n);
        k_dot<double><<<g, kBlock, 0, s>>>(n, (const double *)x, (const double *)y, (double *)ws.partials,
                                           ws.counters, (double *)result, 0);
    } else {
        int g = grid_for(k_dot<float>, 0, n);
        k_dot<float><<<g, kBlock, 0, s>>>(n, (const float *)x, (const float *)y, (float *)ws.partials, ws.counters,
                                          (float *)result, 0);
    }
    return check_launch("k_dot");
}

int mpk_norm2(int32_t dtype, int64_t n, const void *x, void *result, void *ws_, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Ws ws = carve(ws_);
    if (dtype == MPK_F64) {
        int g = grid_for(k_dot<double>, 0, n);
        k_dot<double><<<g, kBlock, 0, s>>>(n, (const double *)x, (const double *)x, (double *)ws.partials,
                                           ws.counters, (double *)result, 1);
    } else {
        int g = grid_for(k_dot<float>, 0, n);
        k_dot<float><<<g, kBlock, 0, s>>>(n, (const float *)x, (const float *)x, (float *)ws.partials, ws.counters,
                                          (float *)result, 1);
    }
    return check_launch("k_norm2");
}

int mpk_axpy(int32_t dtype, int64_t n, double alpha, const void *x, const void *y, void *out, void *stream) {
    if (n == 0) return MPK_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == MPK_F64) {
        int g = grid_for(k_axpy<double>, 0, n);
        k_axpy<double><<<g, kBlock, 0, s>>>(n, alpha, (const double *)x, (const double *)y, (double *)out);
    } else {
        int g = grid_for(k_axpy<float>, 0, n);
        k_axpy<float><<<g, kBlock, 0, s>>>(n, (float)alpha, (const float *)x, (const float *)y, (float *)out);
    }
    return check_launch("k_axpy");
}

int mpk_scale(int32_t dtype, int64_t n, double alpha, const void *x, void *out, void *stream) {
    return mpk_axpy(dtype, n, alpha, x, nullptr, out, stream);
}

int mpk_cgs2_append(int32_t dtype, int64_t n, int64_t ld, int32_t count, void *V, const void *w, int32_t rule,
                    void *coeffs, void *out, int32_t *appended_dev, void *tmp, void *ws_, void *stream) {
    if (count < 1) return fail(MPK_EARG, "basis must hold at least one vector");
    cudaStream_t s = (cudaStream_t)stream;
    Ws ws = carve(ws_);
    if (dtype == MPK_F64)
        return cgs2_append_t<double>(n, ld, count, (double *)V, (const double *)w, rule, (double *)coeffs,
                                     (double *)out, appended_dev, (double *)tmp, ws, s);
    return cgs2_append_t<float>(n, ld, count, (float *)V, (const float *)w, rule, (float *)coeffs, (float *)out,
                                appended_dev, (float *)tmp, ws, s);
}

int mpk_cycle_run(const mpk_cycle_desc *d, void *stream) {
    if (!d || !d->A || !d->V || !d->ctl || !d->ws || !d->hess || !d->work) return fail(MPK_EARG, "null argument");
    if (d->ld < d->n) return fail(MPK_EARG, "ld < n");
    cudaStream_t s = (cudaStream_t)stream;
    g_prof_on = (d->flags & 1) != 0;
    int rc = d->dtype == MPK_F64 ? run_cycle<double>(d, s) : run_cycle<float>(d, s);
    g_prof_on = false;
    return rc;
}

int mpk_residual(const mpk_matrix *A, const void *b, const void *x, void *r, void *sums, float *r_low,
                 float *sums_low, void *ws_, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Ws ws = carve(ws_);
    if (A->dtype == MPK_F64)
        return launch_residual<double>(A, (const double *)b, (const double *)x, (double *)r, (double *)sums, r_low,
                                       sums_low, ws, s);
    return launch_residual<float>(A, (const float *)b, (const float *)x, (float *)r, (float *)sums, nullptr, nullptr,
                                  ws, s);
}

int mpk_ir_update(int64_t n, double *x, const float *u, int32_t *changed, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int g = grid_for(k_ir_update, 0, n);
    // the "x moved" flag is this refinement's: cleared stream-ordered here
    if (changed) {
        cudaError_t e = cudaMemsetAsync(changed, 0, sizeof(int32_t), s);
        if (e != cudaSuccess) return fail(MPK_ELAUNCH, cudaGetErrorString(e));
    }
    k_ir_update<<<g, kBlock, 0, s>>>(n, x, u, changed);
    return check_launch("k_ir_update");
}

int mpk_precond_apply(const mpk_precond *M, const void *v, void *out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (M->dtype == MPK_F64) return apply_precond_t<double>(M, (const double *)v, (double *)out, nullptr, s);
    return apply_precond_t<float>(M, (const float *)v, (float *)out, nullptr, s);
}

int mpk_lsq_init(int32_t dtype, int32_t m, double gamma, double norm_scale, void *hess, mpk_cycle_ctl *ctl,
                 void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == MPK_F64)
        k_lsq_init<double><<<1, 32, 0, s>>>(hess_view<double>(hess, m), ctl, gamma, norm_scale);
    else
        k_lsq_init<float><<<1, 32, 0, s>>>(hess_view<float>(hess, m), ctl, gamma, norm_scale);
    return check_launch("k_lsq_init");
}

int mpk_lsq_update(int32_t dtype, int32_t m, int32_t j, const void *coeffs, const void *beta, void *hess,
                   mpk_cycle_ctl *ctl, void *ws_, void *stream) {
    if (j < 1 || j > m) return fail(MPK_EARG, "column index out of range");
    cudaStream_t s = (cudaStream_t)stream;
    Ws ws = carve(ws_);
    const StepParams p{j - 1, m, 0.0, -1.0, 0};
    const size_t smem = (size_t)(3 * m + 1) * (dtype == MPK_F64 ? 8 : 4);
    if (dtype == MPK_F64)
        k_lsq_update<double><<<1, 32, smem, s>>>((const double *)coeffs, (const double *)beta, (double *)ws.sums,
                                                 hess_view<double>(hess, m), ctl, p);
    else
        k_lsq_update<float><<<1, 32, smem, s>>>((const float *)coeffs, (const float *)beta, (float *)ws.sums,
                                                hess_view<float>(hess, m), ctl, p);
    return check_launch("k_lsq_update");
}

int mpk_lsq_solve(int32_t dtype, int32_t m, int32_t k, void *hess, mpk_cycle_ctl *ctl, void *stream) {
    if (k < 1 || k > m) return fail(MPK_EARG, "k out of range");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == MPK_F64)
        k_lsq_solve<double><<<1, 32, (size_t)(m + 1) * 8, s>>>(hess_view<double>(hess, m), ctl,
                                                              std::ldexp(1.0, -53), k);
    else
        k_lsq_solve<float><<<1, 32, (size_t)(m + 1) * 4, s>>>(hess_view<float>(hess, m), ctl,
                                                             std::ldexp(1.0, -24), k);
    return check_launch("k_lsq_solve");
}

int mpk_block_lu(const mpk_matrix *A, int32_t k, void *lu, int32_t *piv, void *minpiv, double *thr, int32_t *bad,
                 void *stream) {
    if (!A || A->kind != MPK_CSR || !lu || !piv || !minpiv || !thr || !bad) return fail(MPK_EARG, "null argument");
    if (k < 1 || k > 64) return fail(MPK_EUNSUPPORTED, "block Jacobi block size must be 1..64 on the device");
    if (A->n == 0) return MPK_OK;
    cudaStream_t s = (cudaStream_t)stream;
    auto go = [&](auto tag) -> int {
        using T = decltype(tag);
        const CsrOp<T> op = make_csr<T>(A);
        const double u = sizeof(T) == 8 ? 1.1102230246251565e-16 : 5.9604644775390625e-08;
        const size_t smem = (size_t)kLuWarps * k * k * sizeof(T);
        cudaFuncSetAttribute(k_block_lu<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t nb = (A->n + k - 1) / k;
        int64_t g = (nb + kLuWarps - 1) / kLuWarps;
        if (g > 8 * (int64_t)sm_count_cached()) g = 8 * (int64_t)sm_count_cached();
        k_block_lu<T><<<(int)g, kLuWarps * 32, smem, s>>>(op, k, u, (T *)lu, piv, (T *)minpiv, thr, bad);
        return check_launch("k_block_lu");
    };
    return A->dtype == MPK_F64 ? go(double{}) : go(float{});
}

int mpk_stencil_assemble(const mpk_matrix *S, int64_t *row_ptr, int32_t *col_idx, double *values, void *work,
                         void *stream) {
    if (!S || S->kind != MPK_STENCIL || !row_ptr || !col_idx || !values || !work)
        return fail(MPK_EARG, "null argument or not a stencil");
    if (S->row0 != 0) return fail(MPK_EARG, "assembly of a whole matrix only (row0 = 0)");
    cudaStream_t s = (cudaStream_t)stream;
    const StencilOp<double> op = make_stencil<double>(S);
    const int64_t n = op.n;
    if (n == 0) return MPK_OK;
    int32_t *cnt = (int32_t *)work;
    int64_t *bsum = (int64_t *)((char *)work + ((n * 4 + 255) / 256) * 256);
    const int64_t nb = (n + kScanChunk - 1) / kScanChunk;
    int g = grid_for(k_stencil_count<double>, 0, n);
    k_stencil_count<double><<<g, kBlock, 0, s>>>(op, cnt);
    k_scan_local<<<(unsigned)nb, kScanThreads, 0, s>>>(cnt, n, row_ptr, bsum);
    k_scan_blocks<<<1, kScanThreads, 0, s>>>(bsum, nb);
    k_scan_add<<<g, kBlock, 0, s>>>(row_ptr, n, bsum);
    k_stencil_fill<double><<<g, kBlock, 0, s>>>(op, row_ptr, col_idx, values);
    return check_launch("k_stencil_fill");
}

int64_t mpk_stencil_assemble_ws_bytes(int64_t n) {
    return ((n * 4 + 255) / 256) * 256 + ((n + kScanChunk - 1) / kScanChunk) * 8 + 256;
}

int64_t mpk_launch_count(void) { return (int64_t)g_launches; }
const char *mpk_last_cycle_kernel(void) { return g_last_cycle; }

int mpk_prof_reset(void) {
    prof_drain(true);
    for (int i = 0; i < kProfClasses; ++i) {
        g_prof_ms[i] = 0;
        g_prof_cnt[i] = 0;
        g_prof_bytes[i] = 0;
    }
    return MPK_OK;
}

int64_t mpk_comm_part_bytes(int32_t dtype) {
    // cycle partials, then the per-restart scalar slot table (comm.cuh)
    return comm_part_core(dtype) + (int64_t)kMaxRanks * kCommScalBytes;
}

int mpk_can_access_peer(int32_t dev, int32_t peer) {
    if (dev == peer) return 1;
    int ok = 0;
    cudaError_t e = cudaDeviceCanAccessPeer(&ok, dev, peer);
    if (e != cudaSuccess) return fail(MPK_ELAUNCH, cudaGetErrorString(e));
    return ok ? 1 : 0;
}

int mpk_comm_push_rows(const mpk_comm *c, int32_t dtype, int64_t n, const void *x, void *stream) {
    CommView v;
    if (int rc = comm_view(c, dtype, v)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t g = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count_cached() * 4;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    if (dtype == MPK_F64) k_comm_push<double><<<(int)g, 256, 0, s>>>(v, n, (const double *)x);
    else k_comm_push<float><<<(int)g, 256, 0, s>>>(v, n, (const float *)x);
    return check_launch("k_comm_push");
}

int mpk_comm_reduce_ctl(const mpk_comm *c, int32_t dtype, void *slot32, int32_t rn2_dtype, int32_t bn2_dtype,
                        void *stream) {
    CommView v;
    if (int rc = comm_view(c, dtype, v)) return rc;
    if ((uintptr_t)slot32 % 16) return fail(MPK_EARG, "scalar slot must be 16-byte aligned");
    k_comm_reduce<<<1, 32, 0, (cudaStream_t)stream>>>(v, (char *)slot32, rn2_dtype == MPK_F64,
                                                       bn2_dtype == MPK_F64);
    return check_launch("k_comm_reduce");
}

int mpk_dev_alloc(int64_t bytes, void **ptr) {
    if (!ptr || bytes <= 0) return fail(MPK_EARG, "mpk_dev_alloc: bad arguments");
    cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
    if (e != cudaSuccess) return fail(MPK_ELAUNCH, cudaGetErrorString(e));
    e = cudaMemset(*ptr, 0, (size_t)bytes);
    if (e != cudaSuccess) return fail(MPK_ELAUNCH, cudaGetErrorString(e));
    return MPK_OK;
}

int mpk_dev_free(void *ptr) {
    cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? MPK_OK : fail(MPK_ELAUNCH, cudaGetErrorString(e));
}

int mpk_ipc_get(const void *ptr, void *handle64) {
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(ptr));
    if (e != cudaSuccess) return fail(MPK_ELAUNCH, cudaGetErrorString(e));
    memcpy(handle64, &h, sizeof(h));
    return MPK_OK;
}

int mpk_ipc_open(const void *handle64, void **ptr) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? MPK_OK : fail(MPK_ELAUNCH, cudaGetErrorString(e));
}

int mpk_ipc_close(void *ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    return e == cudaSuccess ? MPK_OK : fail(MPK_ELAUNCH, cudaGetErrorString(e));
}

int mpk_fused_prof_read(uint64_t *out, int32_t nctas) {
    if (nctas > kFMaxCtas) nctas = kFMaxCtas;
    cudaError_t e = cudaMemcpyFromSymbol(out, g_fused_prof, sizeof(uint64_t) * kProfSlots * nctas);
    if (e != cudaSuccess) return fail(MPK_ELAUNCH, cudaGetErrorString(e));
    return MPK_OK;
}

int mpk_prof_read(double *ms, int64_t *counts, double *bytes, int32_t nclasses) {
    prof_drain(true);
    for (int i = 0; i < nclasses && i < kProfClasses; ++i) {
        ms[i] = g_prof_ms[i];
        counts[i] = g_prof_cnt[i];
        bytes[i] = g_prof_bytes[i];
    }
    return MPK_OK;
}

}  // extern "C"
