// Host runtime and C-ABI of the DET engine.  See include/det_api.h.
//
// A context owns one CUDA stream, the map topology, a batch of cartograms and
// all device buffers.  det_run() keeps the whole iteration loop on the device:
// one iteration = k_sat1 -> k_sat2 -> k_sat3 -> k_region -> k_row -> k_ctrl per
// frame group; 16 iterations of every group are captured into one CUDA graph,
// the groups as parallel branches (fork/join).  Kernels of finished cartograms
// exit on their device-side `active` flag, and the host only polls the flags
// once per graph launch.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/det_api.h"
#include "det_common.cuh"
#include "det_ctrl.cuh"
#include "det_raster.cuh"
#include "det_sat.cuh"
#include "det_metrics.cuh"
#include "det_mapping.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_select.cuh>

using namespace det;

namespace {

// DET_GUARD=1 (debug mode; compute-sanitizer is not available on the GPU pool): every device
// buffer is allocated with a 4 KB guard zone on each side filled with 0xA5, and its contents are
// poisoned with 0xFF bytes (NaN doubles / -1 ints) instead of left as whatever cudaMalloc returns.
// det_debug_guard_check() compares every live guard zone with the pattern: a kernel that writes
// before or after one of its buffers shows up as a corrupted guard, and a kernel that reads a
// buffer before anything wrote it sees NaN / -1 and fails the parity tests.
constexpr size_t kGuard = 4096;
constexpr unsigned char kGuardByte = 0xA5;
struct GuardAlloc {
    char* raw;
    size_t bytes;
    int device;
};
static std::mutex g_guard_mu;
// guard mode only: its allocations poison memory through the legacy stream and synchronise the
// device, which would invalidate a graph capture running on another thread (one context per
// steering session) -- captures and guard allocations exclude each other
static std::recursive_mutex g_guard_capture_mu;
static std::vector<GuardAlloc> g_guard_live;
static long long g_guard_bad_freed = 0;  // corrupted guards found when a buffer was released
static bool guard_mode() {
    static const int on = [] {
        const char* e = getenv("DET_GUARD");
        return e && atoi(e) != 0 ? 1 : 0;
    }();
    return on != 0;
}
static bool guard_intact(const GuardAlloc& g) {
    std::vector<unsigned char> h(2 * kGuard);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(g.device);
    cudaDeviceSynchronize();
    bool ok = cudaMemcpy(h.data(), g.raw, kGuard, cudaMemcpyDeviceToHost) == cudaSuccess &&
              cudaMemcpy(h.data() + kGuard, g.raw + kGuard + g.bytes, kGuard, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaSetDevice(prev);
    for (size_t i = 0; ok && i < h.size(); ++i) ok = h[i] == kGuardByte;
    return ok;
}
static cudaError_t dev_alloc(void** out, size_t bytes) {
    if (!guard_mode()) return cudaMalloc(out, bytes);
    std::lock_guard<std::recursive_mutex> cap(g_guard_capture_mu);
    char* raw = nullptr;
    cudaError_t e = cudaMalloc(&raw, bytes + 2 * kGuard);
    if (e != cudaSuccess) return e;
    cudaMemset(raw, kGuardByte, kGuard);
    cudaMemset(raw + kGuard, 0xFF, bytes);
    cudaMemset(raw + kGuard + bytes, kGuardByte, kGuard);
    e = cudaDeviceSynchronize();
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guard_live.push_back({raw, bytes, dev});
    *out = raw + kGuard;
    return e;
}
static void dev_free(void* p) {
    if (!guard_mode()) {
        cudaFree(p);
        return;
    }
    char* raw = static_cast<char*>(p) - kGuard;
    std::lock_guard<std::recursive_mutex> cap(g_guard_capture_mu);
    std::lock_guard<std::mutex> lk(g_guard_mu);
    for (size_t i = 0; i < g_guard_live.size(); ++i) {
        if (g_guard_live[i].raw != raw) continue;
        if (!guard_intact(g_guard_live[i])) ++g_guard_bad_freed;
        g_guard_live.erase(g_guard_live.begin() + (long)i);
        break;
    }
    cudaFree(raw);
}

template <typename T>
struct DVec {
    T* p = nullptr;
    size_t n = 0;
    DVec() = default;
    DVec(const DVec&) = delete;
    DVec& operator=(const DVec&) = delete;
    ~DVec() { release(); }
    void release() {
        if (p) dev_free(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count) {  // exact-or-larger, contents undefined
        if (p && count <= n) return cudaSuccess;
        release();
        void* q = nullptr;
        cudaError_t e = dev_alloc(&q, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) {
            p = static_cast<T*>(q);
            n = std::max<size_t>(count, 1);
        }
        return e;
    }
};

#ifndef DET_GRAPH_ITERS
#define DET_GRAPH_ITERS 16
#endif
constexpr int kGraphIters = DET_GRAPH_ITERS;  // iterations per graph launch (32: +0.?% at 296 frames, more gated launches for a lone cartogram)

}  // namespace

struct det_ctx {
    int device = 0, k = 10, n = 1024, f64 = 0, s64 = 0, H = 8;  // f64: float64 field; s64: float64 vertex state
    bool bitmap_raster = false;  // k_region<..., true>: scanlines with more crossings than its toggle window
    bool raster_ro = true;       // launches without advect use k_region<..., ADV=false> (DET_RASTER_RO=0: off)
    cudaStream_t stream = nullptr;
    std::string err;
    // topology
    int R = 0, n_rows = 0, n_rings = 0;
    std::vector<int> h_ring_start, h_region_ring0;
    DVec<double2> xy_rows;  // the loaded vertex rows, device resident (start geometry of every batch)
    DVec<int> region_row0, region_rank, rank_region, ring_start, region_ring0, row_next;
    // batch
    int B = 0, cap = 64, nb = 0, trace_cap = 0;
    // pos0 (the state rows, advected in place) and best hold float2 rows on the float32-field
    // path (sized as double2 either way);
    // rows64 is the widened copy of a float state handed to the read-back / area paths
    DVec<double2> pos_init, pos0, best, rows64;
    DVec<int> labels, cnt_acc, cnt_state, rowcnt, maxspan, rowdone;
    DVec<unsigned long long> spans;
    DVec<float> lutf;
    DVec<double> lut, stats, weights, rerr, cs, dgc, adc, rt, csX, dgXc, adSc, csT, dgT, adT, rowfull, tab, trace;
    DVec<char> uf;
    DVec<Carto> st;
    DVec<Params> prm;
    std::vector<Params> h_prm;
    std::vector<Carto> h_st;
    bool params_set = false, ran = false, bench_mode = false, h_fixed = false;
    // stage buffers
    DVec<double> dense, ch8, uf64, pts_in, pts_out;
    DVec<unsigned long long> clampbuf;
    // graph
    cudaGraphExec_t gexec = nullptr;
    bool g_valid = false;
    int groups = 8;  // graph branches (clamped to the batch); 1/2/4/8 measured 41.5/42.4/43.9/44.2k it/s
    bool sep_ctrl = true;  // control step as its own kernel (DET_SEP_CTRL=0: k_row's last CTA)
    bool sat1w = true;  // float32 field: barrier-free k_sat1w (DET_SAT1W=0: k_sat1)
    bool sat3w = true;  // float64 field: barrier-free k_sat3w with k_sat1w's slice tables (DET_SAT3W=0: k_sat3)
    bool sat3x = true;  // k_sat3w as k_sat3x (edge records prefixed per band, rows unrolled 4x; DET_SAT3X=0: k_sat3w)
    bool sat1x = true;  // k_sat1w (float64, slice tables) as k_sat1x (DET_SAT1X=0: k_sat1w)
    bool split_adv = false;  // float32 state: advect as the flat k_advect_rows (DET_SPLIT_ADVECT=1); 48.6k vs 51.4k fused
    // float64: advect once per unique vertex (k_advect_uniq64) + the raster-only k_region; valid while
    // every frame's start rows keep the loaded map's shared vertices bit-identical (ua_ok)
    bool uniq_adv = true;
    bool ua_ok = false;
    int n_uniq = 0;
    DVec<int> uq_row0, uq_off, uq_rows, row_uniq, uq_flag;
    DVec<double2> upos, ubest;  // unique-vertex state of the graph iterations (see k_uq_gather)
    bool uq_state = true;       // DET_UQ_STATE=0: the graph iterations advect the rows (k_advect_uniq64)
    bool g_uqs = false;
    DVec<unsigned char> uq_band0, uq_band1;  // band-fused advect: per-vertex band bytes, by iteration parity
    int uq_bstride = 0;
    // DET_FUSE_ADVECT=1 (experiment, off): k_sat3x advects a band's vertices after its sweep.  Correct
    // (bit-identical, tested) but slower: 44.0k vs 61.6k it/s -- with 16 warps per SM the band CTA
    // serialises the position -> texel round trips that the flat advect hides with 53 warps per SM
    bool fuse_adv = false;
    bool g_fa = false;
    std::vector<int> h_uq_off, h_uq_rows, h_uq_row0, h_row_uniq;
    std::vector<double> h_xy_prev;  // the rows the unique-vertex table was built from
    bool g_ua = false;
    int g_nuniq = 0;
    const void* g_uq = nullptr;  // the unique-vertex arrays and count are kernel arguments the graph bakes in
    const void* g_uq0 = nullptr;
    Topo g_topo;  // launch signature the graph was captured with
    Bufs g_bufs;
    int g_groups = 0;
    std::vector<cudaStream_t> gstreams;
};

#define CK(expr)                                                                   \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ctx->err = std::string(#expr) + ": " + cudaGetErrorString(_e);         \
            return DET_E_CUDA;                                                     \
        }                                                                          \
    } while (0)

static int fail(det_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}


static Topo make_topo(det_ctx* c) {
    Topo t;
    memset(&t, 0, sizeof(t));
    t.n_rows = c->n_rows;
    t.R = c->R;
    t.region_row0 = c->region_row0.p;
    t.ring_start = c->ring_start.p;
    t.region_ring0 = c->region_ring0.p;
    t.region_rank = c->region_rank.p;
    t.rank_region = c->rank_region.p;
    t.row_next = c->row_next.p;
    t.row_uniq = c->row_uniq.p;
    return t;
}

static Bufs make_bufs(det_ctx* c) {
    Bufs d;
    memset(&d, 0, sizeof(d));
    d.B = c->B; d.n = c->n; d.k = c->k; d.cap = c->cap; d.H = c->H; d.nb = c->nb;
    d.nn = (size_t)c->n * c->n;
    d.pos0 = c->pos0.p; d.best = c->best.p;
    d.upos = c->upos.p; d.ubest = c->ubest.p; d.uq_flag = c->uq_flag.p; d.n_uniq = c->n_uniq;
    if (c->fuse_adv) { d.uq_band[0] = c->uq_band0.p; d.uq_band[1] = c->uq_band1.p; }  // (null: k_uq_gather skips the band bytes)
    d.uq_bstride = c->uq_bstride;
    d.labels = c->labels.p; d.cnt_acc = c->cnt_acc.p; d.cnt_state = c->cnt_state.p;
    d.spans = c->spans.p; d.rowcnt = c->rowcnt.p; d.maxspan = c->maxspan.p; d.rowdone = c->rowdone.p;
    d.lut = c->lut.p; d.lutf = c->lutf.p; d.stats = c->stats.p; d.weights = c->weights.p; d.rerr = c->rerr.p;
    d.uf = c->uf.p;
    d.cs = c->cs.p; d.dgc = c->dgc.p; d.adc = c->adc.p; d.rt = c->rt.p;
    d.csX = c->csX.p; d.dgXc = c->dgXc.p; d.adSc = c->adSc.p;
    d.csT = c->csT.p; d.dgT = c->dgT.p; d.adT = c->adT.p; d.rowfull = c->rowfull.p; d.tab = c->tab.p;
    d.st = c->st.p; d.prm = c->prm.p; d.trace = c->trace.p; d.trace_cap = c->trace_cap;
    return d;
}

// ----------------------------- launch helpers ---------------------------------
// Dynamic shared-memory opt-in.  The attribute is process-wide per kernel, so contexts on other
// threads (one per steering session) must never lower it under a launch being captured: every
// caller sets the same value, the device's opt-in maximum minus the kernel's static shared memory
// (idempotent, race-free).
template <typename F>
static void smem_optin(F fn) {
    static int max_optin = [] {
        int dev = 0, v = 48 * 1024;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        return v;
    }();
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, fn) != cudaSuccess) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin - (int)a.sharedSizeBytes);
}

#ifndef DET_SAT3_CPT
#define DET_SAT3_CPT 4  // k_sat3 columns per thread on the float32 path
#endif
static int skip_mask();
// graph iterations on the unique-vertex state: float64, every shared vertex bit-identical in the
// start rows, the plain (non-bitmap) raster
static bool uqs_on(const det_ctx* c) {
    return c->f64 && c->uniq_adv && c->ua_ok && c->uq_state && !c->bitmap_raster && !(skip_mask() & 4);
}

// band-fused advect: the unique-vertex state, k_sat3x with one CTA per band row (n = 512 or 1024),
// band ids in a byte
static bool fa_on(const det_ctx* c) {
    return uqs_on(c) && c->fuse_adv && c->sat1w && c->sat3w && c->sat3x && (c->n == 512 || c->n == 1024) &&
           c->H < 128 && c->nb < 254 && !(skip_mask() & 2);
}

// Diagnostics only (timing experiments, results invalid): DET_SKIP bit mask of iteration stages
// left out of the captured graph -- 1 band sums + carries (k_sat1w, k_sat2p), 2 k_sat3,
// 4 advect + raster (k_region), 8 paint + control step (k_row, k_ctrl).
static int skip_mask() {
    static const int m = [] { const char* e = getenv("DET_SKIP"); return e ? atoi(e) : 0; }();
    return m;
}

template <int CPT, int NT>
static void launch_sat_cfg(det_ctx* c, const Topo& T, const Bufs& D, const SatSrc& S, int gate, int src, int out,
                           bool u64, int B, int fa = -1) {
    const int n = c->n, H = c->H, R = c->R;
    const dim3 gb(c->nb, B);
    // float32 in-band arithmetic only for the float32 field from labels; float64 otherwise
    const bool f32 = (src == SRC_LABELS && out == OUT_U && !u64);
    const size_t sa = f32 ? sizeof(float) : sizeof(double);
    // the residual-density LUT goes to shared memory when it fits in 48 KB
    const bool luts = src == SRC_LABELS && (size_t)lut_smem_len(R) * sa <= 48 * 1024;
    const size_t lut_b = luts ? (size_t)lut_smem_len(R) * sa : 0;
    // k_sat3's label ring (lab_kp rows of NT*CPT ints; see RING in k_sat3)
    const size_t ring_b = (src == SRC_LABELS && out == OUT_U && (f32 || CPT * NT <= 4096))
                              ? (size_t)lab_kp(CPT * NT) * NT * CPT * sizeof(int) : 0;
    const size_t ring1_b = (src == SRC_LABELS && f32) ? (size_t)lab_kp1(CPT * NT) * NT * CPT * sizeof(int) : 0;
    const size_t smem1 = ((size_t)2 * (n + H - 1) + (size_t)H * (NT / 32)) * sa + ring1_b + 16;
#define DET_SAT1(SRC_, A_, L_)                                                                               \
    do {                                                                                                     \
        auto fn = k_sat1<CPT, NT, SRC_, A_, L_>;                                                             \
        smem_optin(fn);                                                                                      \
        fn<<<gb, NT, smem1, c->stream>>>(T, D, S, gate);                                                     \
    } while (0)
    // barrier-free sweep, one TMA ring per warp slice (k_sat1w; DET_SAT1W_CPT columns per thread
    // where the band kernels use 4)
    constexpr int CPT1 = (CPT == 4 && NT * 4 / DET_SAT1W_CPT <= 1024 && NT * 4 / DET_SAT1W_CPT >= 32) ? DET_SAT1W_CPT : CPT;
    constexpr int NT1 = NT * CPT / CPT1;
    const bool skip12 = src == SRC_LABELS && out == OUT_U && (skip_mask() & 1);
    const bool skip3 = src == SRC_LABELS && out == OUT_U && (skip_mask() & 2);
    const bool sat1w_ok = src == SRC_LABELS && out == OUT_U && c->sat1w && n % (32 * CPT1) == 0 && (f32 || n <= 4096);
    // float64 field: the barrier-free k_sat3w (128-column warp slices, band height below the slice
    // width) fed by k_sat1w's slice tables
    const bool w3 = sat1w_ok && !f32 && c->sat3w && CPT1 == 4 && n >= 512 && H < 32 * CPT1;
    if (skip12) {
    } else if (w3) {
        constexpr int NW = NT1 / 32, KP = lab_kp1(CPT1 * NT1);
        size_t smem1w = ((size_t)2 * (n + H - 1) + (size_t)4 * H * NW) * sa + 16 +
                        (size_t)NW * KP * 32 * CPT1 * sizeof(int);
        const bool l1 = DET_SAT1W_LUTS && (size_t)lut_smem_len(R) * sa <= 48 * 1024;
        if (l1) smem1w += (size_t)lut_smem_len(R) * sa;
        bool done1 = false;
        if constexpr (CPT1 == 4 && NT1 <= 512) {
            if (c->sat1x) {  // rows unrolled 4x over an 8-slot ring, dg/ad aliased (DET_SAT1X=0: k_sat1w)
                const size_t smem1x = (size_t)4 * H * NW * sa + (size_t)NW * 8 * 32 * CPT1 * sizeof(int) +
                                      (l1 ? (size_t)lut_smem_len(R) * sa : 0);
                auto fx = l1 ? k_sat1x<NT1, true> : k_sat1x<NT1, false>;
                smem_optin(fx);
                fx<<<gb, NT1, smem1x, c->stream>>>(T, D, gate);
                done1 = true;
            }
        }
        if (!done1) {
            auto fn = l1 ? k_sat1w<CPT1, NT1, true, double, true> : k_sat1w<CPT1, NT1, false, double, true>;
            smem_optin(fn);
            fn<<<gb, NT1, smem1w, c->stream>>>(T, D, gate);
        }
    } else if (sat1w_ok) {
        // barrier-free band sums in the field's arithmetic type (float32 or float64)
        constexpr int NW = NT1 / 32, KP = lab_kp1(CPT1 * NT1);
        size_t smem1w = ((size_t)2 * (n + H - 1) + (size_t)3 * H * NW) * sa + 16 +
                        (size_t)NW * KP * 32 * CPT1 * sizeof(int);
        const bool l1 = DET_SAT1W_LUTS && (size_t)lut_smem_len(R) * sa <= 48 * 1024;
        if (l1) smem1w += (size_t)lut_smem_len(R) * sa;
        if (f32) {
            auto fn = l1 ? k_sat1w<CPT1, NT1, true, float> : k_sat1w<CPT1, NT1, false, float>;
            smem_optin(fn);
            fn<<<gb, NT1, smem1w, c->stream>>>(T, D, gate);
        } else {
            auto fn = l1 ? k_sat1w<CPT1, NT1, true, double> : k_sat1w<CPT1, NT1, false, double>;
            smem_optin(fn);
            fn<<<gb, NT1, smem1w, c->stream>>>(T, D, gate);
        }
    } else if (src == SRC_LABELS) {
        // k_sat1 gathers the LUT through L1 (__ldg): staging it per CTA measured slower there
        if (f32) DET_SAT1(SRC_LABELS, float, false);
        else DET_SAT1(SRC_LABELS, double, false);
    } else {
        DET_SAT1(SRC_DENSE, double, false);
    }
#undef DET_SAT1
    const int lanes = n + 2 * (2 * n - 1);
    if (skip12) {
    } else if (src == SRC_LABELS && out == OUT_U)  // band carries split over the warps of a CTA (one memory round trip)
        k_sat2p<<<dim3((lanes + 31) / 32 + 1, B), 32 * SAT2_PARTS, 0, c->stream>>>(D, gate);
    else
        k_sat2<<<dim3((lanes + SAT2_THREADS - 1) / SAT2_THREADS + 1, B), SAT2_THREADS, 0, c->stream>>>(D, gate);
    const size_t smem = ((size_t)3 * (n + H) + 3 * H + (H & 1)) * sa + lut_b + ring_b + 16;
#define DET_SAT3(SRC_, UT_, OUT_, L_)                                                                        \
    do {                                                                                                     \
        auto fn = k_sat3<CPT, NT, SRC_, UT_, OUT_, UT_, L_>;                                                 \
        smem_optin(fn);                                                                                      \
        fn<<<gb, NT, smem, c->stream>>>(T, D, S, gate);                                                      \
    } while (0)
    if (skip3) {
    } else if (w3) {
        // CTAs of up to 8 warp slices (1024 columns) per band
        constexpr int NTW = NT * CPT >= 1024 ? 256 : NT;
        constexpr int NWC = NTW / 32, W = 32 * CPT;
        constexpr int KPW = lab_kp(W * NWC) > 4 ? 4 : lab_kp(W * NWC);
        const int WN = NWC * W + H, PW = (WN + 3) / 4 + 1;  // phase-split windows (k_sat3w)
        const size_t smemw = ((size_t)3 * 4 * PW + 3 * H + (H & 1) + (size_t)4 * (NWC + 2) * H +
                              (size_t)NWC * (H + 1) + ((NWC * (H + 1)) & 1)) * sizeof(double) +
                             lut_b + (size_t)NWC * KPW * W * sizeof(int) + 16;
        if constexpr (CPT == 4) {
            if (c->sat3x) {  // loop-invariant edge records + 4x unrolled rows (DET_SAT3X=0: k_sat3w)
                const size_t smemx = ((size_t)3 * 4 * sat3x_phase_len(NWC) + (size_t)NWC * H * 6) * sizeof(double) +
                                     lut_b + (size_t)NWC * 4 * W * sizeof(int) + 16;
                if (fa >= 0 && n == NWC * W) {  // band-fused advect (one CTA per band row)
                    auto fa_k = luts ? k_sat3x<NTW, true, true> : k_sat3x<NTW, false, true>;
                    smem_optin(fa_k);
                    fa_k<<<dim3(c->nb, B, 1), NTW, smemx, c->stream>>>(T, D, gate, fa, c->uq_off.p);
                    return;
                }
                auto fx = luts ? k_sat3x<NTW, true> : k_sat3x<NTW, false>;
                smem_optin(fx);
                fx<<<dim3(c->nb, B, n / (NWC * W)), NTW, smemx, c->stream>>>(T, D, gate, -1, nullptr);
                return;
            }
        }
        auto fn = luts ? k_sat3w<CPT, NTW, true> : k_sat3w<CPT, NTW, false>;
        smem_optin(fn);
        fn<<<dim3(c->nb, B, n / (NWC * W)), NTW, smemw, c->stream>>>(T, D, gate);
    } else if (out == OUT_CH8) {
        if (src == SRC_LABELS) {
            if (luts) DET_SAT3(SRC_LABELS, double, OUT_CH8, true);
            else DET_SAT3(SRC_LABELS, double, OUT_CH8, false);
        } else {
            DET_SAT3(SRC_DENSE, double, OUT_CH8, false);
        }
    } else if (src == SRC_LABELS) {
        if (u64) {
            if (luts) DET_SAT3(SRC_LABELS, double, OUT_U, true);
            else DET_SAT3(SRC_LABELS, double, OUT_U, false);
        } else {
            // float32 field: DET_SAT3_CPT columns per thread (the ring row and windows are unchanged)
            constexpr int CPT3 = (CPT == 4 && NT * 4 / DET_SAT3_CPT >= 32) ? DET_SAT3_CPT : CPT;
            constexpr int NT3 = NT * CPT / CPT3;
            const size_t ring3_b = (size_t)lab_kp(CPT3 * NT3) * NT3 * CPT3 * sizeof(int);
            const size_t smem3 = ((size_t)3 * (n + H) + 3 * H + (H & 1)) * sa + lut_b + ring3_b + 16;
            auto fn = luts ? k_sat3<CPT3, NT3, SRC_LABELS, float, OUT_U, float, true>
                           : k_sat3<CPT3, NT3, SRC_LABELS, float, OUT_U, float, false>;
            smem_optin(fn);
            fn<<<gb, NT3, smem3, c->stream>>>(T, D, S, gate);
        }
    } else {
        if (u64) DET_SAT3(SRC_DENSE, double, OUT_U, false);
        else DET_SAT3(SRC_DENSE, float, OUT_U, false);
    }
#undef DET_SAT3
}

// band kernels: one CTA per band row-set; CPT columns per thread, NT = n/CPT threads (>= 32)
static void launch_sat(det_ctx* c, const Topo& T, const Bufs& D, const SatSrc& S, int gate, int src, int out, bool u64,
                       int B, int fa = -1) {
    switch (c->n) {
        case 16: case 32: case 64: launch_sat_cfg<2, 32>(c, T, D, S, gate, src, out, u64, B, fa); break;
        case 128: launch_sat_cfg<2, 64>(c, T, D, S, gate, src, out, u64, B, fa); break;
        case 256: launch_sat_cfg<2, 128>(c, T, D, S, gate, src, out, u64, B, fa); break;
        case 512: launch_sat_cfg<4, 128>(c, T, D, S, gate, src, out, u64, B, fa); break;
        case 1024: launch_sat_cfg<4, 256>(c, T, D, S, gate, src, out, u64, B, fa); break;
        case 2048: launch_sat_cfg<4, 512>(c, T, D, S, gate, src, out, u64, B, fa); break;
        case 4096: launch_sat_cfg<4, 1024>(c, T, D, S, gate, src, out, u64, B, fa); break;
        default: launch_sat_cfg<8, 1024>(c, T, D, S, gate, src, out, u64, B, fa); break;
    }
}

// f64_rows: rasterise double2 rows (the start geometry) whatever the context's field type
static void launch_region(det_ctx* c, const Topo& T, const Bufs& D, int mode, int gate, int src,
                          bool f64_rows = false) {
    const dim3 g((c->R + RW_WARPS - 1) / RW_WARPS, c->B);
    if (c->bitmap_raster) {  // a scanline overflowed the toggle window: the parity-bitmap instantiation
        if (c->f64) k_region<double, double, true><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
        else if (c->s64 || f64_rows) k_region<float, double, true><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
        else k_region<float, float, true><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
        return;
    }
    if (!(mode & M_ADVECT) && c->raster_ro) {  // no advect: the raster-only instantiation
        if (c->f64) k_region<double, double, false, false><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
        else if (c->s64 || f64_rows) k_region<float, double, false, false><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
        else k_region<float, float, false, false><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
        return;
    }
    if (c->f64) k_region<double, double><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
    else if (c->s64 || f64_rows) k_region<float, double><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
    else k_region<float, float><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, mode, gate, src);
}

// One iteration's advect + raster: the flat advect kernel then a raster-only k_region (float32
// state), or k_region's fused advect phase.  Returns the number of kernels launched.
static int launch_advect_raster(det_ctx* c, const Topo& T, const Bufs& D, int gate, int region_mode, bool uqs = false,
                                int fa = -1) {
    if (uqs) {  // unique-vertex state (inside a graph launch): coalesced advect, raster through row_uniq
        if (fa >= 0)  // band-fused advect: k_sat3x advected the in-band vertices; the band-straddling ones here
            k_advect_bnd<<<dim3((c->n_uniq + ADV_THREADS - 1) / ADV_THREADS, c->B), ADV_THREADS, 0, c->stream>>>(
                T, D, gate, c->uq_off.p, fa);
        else
        k_advect_uniq64s<<<dim3((c->n_uniq + ADV_THREADS - 1) / ADV_THREADS, c->B), ADV_THREADS, 0, c->stream>>>(
            T, D, gate, c->uq_off.p);
        const dim3 g((c->R + RW_WARPS - 1) / RW_WARPS, c->B);
        k_region<double, double, false, false, true><<<g, RW_WARPS * 32, 0, c->stream>>>(T, D, M_RASTER | M_POSTADV, gate, 0);
        return 2;
    }
    if (c->f64 && c->uniq_adv && c->ua_ok && (region_mode & M_ADVECT)) {
        k_advect_uniq64<<<dim3((c->n_uniq + ADV_THREADS * UQ_PT - 1) / (ADV_THREADS * UQ_PT), c->B), ADV_THREADS, 0,
                          c->stream>>>(
            T, D, gate, c->uq_row0.p, c->uq_off.p, c->uq_rows.p, c->n_uniq);
        if (region_mode & M_RASTER) launch_region(c, T, D, M_RASTER | M_POSTADV, gate, 0);
        return (region_mode & M_RASTER) ? 2 : 1;
    }
    if ((!c->s64 || c->f64) && c->split_adv && (region_mode & M_ADVECT)) {
        const int per = ADV_THREADS * ADV_RPT;
        if (c->f64) k_advect_rows64<<<dim3((T.n_rows + per - 1) / per, c->B), ADV_THREADS, 0, c->stream>>>(T, D, gate);
        else k_advect_rows<<<dim3((T.n_rows + per - 1) / per, c->B), ADV_THREADS, 0, c->stream>>>(T, D, gate);
        if (region_mode & M_RASTER) launch_region(c, T, D, M_RASTER | M_POSTADV, gate, 0);
        return (region_mode & M_RASTER) ? 2 : 1;
    }
    launch_region(c, T, D, region_mode, gate, 0);
    return 1;
}

// ctrl_mode: -1 raster only, 0 loop evaluation, 1 final (best-state) evaluation
static void launch_row(det_ctx* c, const Topo& T, const Bufs& D, int gate, int ctrl_mode) {
    // one warp per texture row; up to 8 rows per CTA within a 64 KB label-row budget
    int rpc = 8;
    while (rpc > 1 && (size_t)rpc * c->n * sizeof(uint32_t) > 64 * 1024) rpc >>= 1;
    rpc = std::min(rpc, c->n);
    const size_t smem = (size_t)rpc * c->n * sizeof(uint32_t);
    smem_optin(k_row);
    k_row<<<dim3((c->n + rpc - 1) / rpc, c->B), rpc * 32, smem, c->stream>>>(T, D, gate, ctrl_mode);
}

// k_row + the loop control step: fused into k_row's last CTA per cartogram, or (sep_ctrl) a
// separate 1024-thread k_ctrl per cartogram after it
static void launch_row_ctrl(det_ctx* c, const Topo& T, const Bufs& D, int gate, int ctrl_mode) {
    if (c->sep_ctrl && ctrl_mode >= 0) {
        launch_row(c, T, D, gate, CTRL_SEPARATE);
        k_ctrl<<<c->B, CTRL_THREADS, 0, c->stream>>>(T, D, ctrl_mode, gate);
    } else {
        launch_row(c, T, D, gate, ctrl_mode);
    }
}

static void enqueue_iteration(det_ctx* c, int b0 = 0, int Bg = -1, cudaStream_t s = nullptr, int uqs = 0,
                              cudaEvent_t after_sat = nullptr) {
    if (Bg < 0) Bg = c->B;
    cudaStream_t keep = c->stream;
    if (s) c->stream = s;
    const Topo T = make_topo(c);
    Bufs D = make_bufs(c);
    D.b0 = b0;
    const int Bsave = c->B;
    c->B = Bg;  // grid.y of every launch below
    SatSrc S;
    memset(&S, 0, sizeof(S));
    const int fa = (uqs & 8) ? ((uqs & 16) ? 1 : 0) : -1;  // band-fused advect: iteration parity
    if (uqs & 1)  // first iteration of a graph launch: rows -> unique-vertex state (+ band bytes)
        k_uq_gather<<<dim3(std::min((c->n_uniq + 255) / 256, 1024), Bg), 256, 0, c->stream>>>(T, D, G_ACTIVE, c->uq_row0.p);
    if ((skip_mask() & 3) != 3) launch_sat(c, T, D, S, G_ACTIVE, SRC_LABELS, OUT_U, c->f64 != 0, Bg, fa);
    if (after_sat) cudaEventRecord(after_sat, c->stream);  // (capture) the staggered neighbour branch starts here
    if (!(skip_mask() & 4)) launch_advect_raster(c, T, D, G_ACTIVE, M_ADVECT | M_RASTER, uqs != 0, fa);
    if (!(skip_mask() & 8)) launch_row_ctrl(c, T, D, G_ACTIVE, 0);
    if (uqs & 4)  // last iteration of a graph launch: unique-vertex state -> rows (+ best rows)
        k_uq_expand<<<dim3(std::min((c->n_rows + 255) / 256, 1024), Bg), 256, 0, c->stream>>>(T, D);
    c->B = Bsave;
    c->stream = keep;
}

static void invalidate_graph(det_ctx* c) {
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
    c->g_valid = false;
}

// Frame groups: the batch is split into up to kGroups contiguous groups whose iteration
// chains are independent branches of one graph, so kernels of different groups overlap.
static int ensure_graph(det_ctx* c) {
    det_ctx* ctx = c;
    {
        // re-capture only when a pointer, shape or the grouping the graph bakes in changed
        const Topo t = make_topo(c);
        const Bufs d = make_bufs(c);
        if (c->g_valid && c->g_groups == c->groups && c->g_ua == (c->uniq_adv && c->ua_ok) && c->g_uqs == uqs_on(c) && c->g_fa == fa_on(c) &&
            c->g_nuniq == c->n_uniq && c->g_uq == c->uq_rows.p && c->g_uq0 == c->uq_row0.p &&
            !memcmp(&t, &c->g_topo, sizeof(t)) &&
            !memcmp(&d, &c->g_bufs, sizeof(d)))
            return DET_OK;
        c->g_topo = t;
        c->g_bufs = d;
        c->g_groups = c->groups;
        c->g_ua = c->uniq_adv && c->ua_ok;
        c->g_uqs = uqs_on(c);
        c->g_fa = fa_on(c);
        c->g_nuniq = c->n_uniq;
        c->g_uq = c->uq_rows.p;
        c->g_uq0 = c->uq_row0.p;
    }
    invalidate_graph(c);
    const int G = std::max(1, std::min(c->groups, c->B));
    while ((int)c->gstreams.size() < G) {
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        c->gstreams.push_back(s);
    }
    cudaEvent_t fork, join[16];
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (int g = 0; g < G; ++g) CK(cudaEventCreateWithFlags(&join[g], cudaEventDisableTiming));
    static const bool stagger = [] { const char* e = getenv("DET_STAGGER"); return e && atoi(e) != 0; }();
    cudaEvent_t stag[16];
    for (int g = 0; g < G; ++g) CK(cudaEventCreateWithFlags(&stag[g], cudaEventDisableTiming));
    cudaGraph_t graph;
    std::unique_lock<std::recursive_mutex> cap(g_guard_capture_mu, std::defer_lock);
    if (guard_mode()) cap.lock();  // (released when this function returns, after EndCapture)
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    CK(cudaEventRecord(fork, c->stream));
    for (int g = 0; g < G; ++g) {
        const int b0 = (int)((long long)c->B * g / G), b1 = (int)((long long)c->B * (g + 1) / G);
        cudaStream_t s = c->gstreams[g];
        CK(cudaStreamWaitEvent(s, fork, 0));
        const bool uqs = uqs_on(c);
        // DET_STAGGER=1 (experiment): odd branches start when their even neighbour has finished its
        // first iteration's band kernels, so the two run out of phase (DRAM-bound kernels of one
        // next to issue-bound kernels of the other)
        const bool lead = stagger && (g % 2 == 0) && g + 1 < G;
        if (stagger && (g % 2 == 1)) CK(cudaStreamWaitEvent(s, stag[g - 1], 0));
        for (int i = 0; i < kGraphIters; ++i)
            enqueue_iteration(c, b0, b1 - b0, s,
                              uqs ? (2 | (i == 0 ? 1 : 0) | (i == kGraphIters - 1 ? 4 : 0) | (fa_on(c) ? 8 : 0) | ((i & 1) ? 16 : 0)) : 0,
                              (lead && i == 0) ? stag[g] : nullptr);
        CK(cudaEventRecord(join[g], s));
        CK(cudaStreamWaitEvent(c->stream, join[g], 0));
    }
    CK(cudaStreamEndCapture(c->stream, &graph));
    cudaError_t e = cudaGraphInstantiate(&c->gexec, graph, 0);
    cudaGraphDestroy(graph);
    cudaEventDestroy(fork);
    for (int g = 0; g < G; ++g) cudaEventDestroy(join[g]);
    for (int g = 0; g < G; ++g) cudaEventDestroy(stag[g]);
    CK(e);
    c->g_valid = true;
    return DET_OK;
}

// ------------------------------- allocation ----------------------------------
static int alloc_spans(det_ctx* ctx) {
    CK(ctx->spans.alloc((size_t)ctx->B * ctx->n * ctx->cap));
    CK(ctx->rowcnt.alloc((size_t)ctx->B * ctx->n));
    CK(cudaMemsetAsync(ctx->rowcnt.p, 0, (size_t)ctx->B * ctx->n * sizeof(int), ctx->stream));
    return DET_OK;
}

static int alloc_sat(det_ctx* ctx, int B) {
    const size_t n = ctx->n, nb = ctx->nb, L = n + ctx->H - 1, M = 2 * n - 1;
    CK(ctx->cs.alloc(B * nb * n));
    CK(ctx->dgc.alloc(B * nb * L));
    CK(ctx->adc.alloc(B * nb * L));
    CK(ctx->rt.alloc(B * n));
    CK(ctx->csX.alloc(B * nb * n));
    CK(ctx->dgXc.alloc(B * nb * n));
    CK(ctx->adSc.alloc(B * nb * (L + 1)));
    CK(ctx->csT.alloc(B * n));
    CK(ctx->dgT.alloc(B * M));
    CK(ctx->adT.alloc(B * M));
    CK(ctx->rowfull.alloc(B * (n + 1)));
    CK(ctx->tab.alloc(B * 4 * n * std::max<size_t>(1, n / 128)));  // nb * 4 * (n/128) slices * H rows
    return DET_OK;
}

#ifndef DET_BAND_FILL
#define DET_BAND_FILL 148  // band CTAs wanted per launch before bands grow taller (2 * 148: B=4 31.3k vs 34.5k, B=8 43.5k vs 44.6k it/s)
#endif
static int auto_band_height(int n, int B) {
    // one band CTA per SM before bands grow taller: tall bands amortise the carries and the
    // per-CTA LUT copy (1024^2: H = 8 for 1-2 frames, 16 for 4, 32 for 8, 64 from 16 frames on)
    int h = 8;
    while (h < 64 && (long long)(n / (2 * h)) * B >= DET_BAND_FILL) h *= 2;
    return std::min(h, n);
}

static int alloc_batch(det_ctx* ctx, int B) {
    const size_t nn = (size_t)ctx->n * ctx->n;
    ctx->B = B;
    if (!ctx->h_fixed) {
        ctx->H = auto_band_height(ctx->n, B);
        ctx->nb = ctx->n / ctx->H;
    }
    CK(ctx->pos_init.alloc((size_t)B * ctx->n_rows));
    CK(ctx->pos0.alloc((size_t)B * ctx->n_rows));
    CK(ctx->best.alloc((size_t)B * ctx->n_rows));
    if (ctx->f64) {
        CK(ctx->upos.alloc((size_t)B * ctx->n_uniq));
        CK(ctx->ubest.alloc((size_t)B * ctx->n_uniq));
        CK(ctx->uq_flag.alloc(B));
        ctx->uq_bstride = (ctx->n_uniq + 15) & ~15;
        if (ctx->fuse_adv) {
        CK(ctx->uq_band0.alloc((size_t)B * ctx->uq_bstride));
        CK(ctx->uq_band1.alloc((size_t)B * ctx->uq_bstride));
        CK(cudaMemsetAsync(ctx->uq_band0.p, 254, (size_t)B * ctx->uq_bstride, ctx->stream));  // pad bytes: no band
        CK(cudaMemsetAsync(ctx->uq_band1.p, 254, (size_t)B * ctx->uq_bstride, ctx->stream));
        }
        CK(cudaMemsetAsync(ctx->uq_flag.p, 0, (size_t)B * sizeof(int), ctx->stream));
    }
    if (!ctx->s64) CK(ctx->rows64.alloc((size_t)B * ctx->n_rows));
    CK(ctx->labels.alloc((size_t)B * nn));
    CK(ctx->cnt_acc.alloc((size_t)B * (ctx->R + 1)));
    CK(ctx->cnt_state.alloc((size_t)B * (ctx->R + 1)));
    CK(ctx->maxspan.alloc((size_t)B));
    CK(ctx->rowdone.alloc((size_t)B));
    CK(cudaMemsetAsync(ctx->rowdone.p, 0, (size_t)B * sizeof(int), ctx->stream));
    CK(ctx->lut.alloc((size_t)B * (ctx->R + 1)));
    CK(ctx->lutf.alloc((size_t)B * (ctx->R + 1)));
    CK(ctx->stats.alloc((size_t)B * ctx->R));
    CK(ctx->weights.alloc((size_t)B * ctx->R));
    CK(ctx->rerr.alloc((size_t)B * ctx->R));
    CK(ctx->uf.alloc((size_t)B * nn * 2 * (ctx->f64 ? 8 : 4)));
    CK(ctx->st.alloc((size_t)B));
    CK(ctx->prm.alloc((size_t)B));
    CK(cudaMemsetAsync(ctx->cnt_acc.p, 0, (size_t)B * (ctx->R + 1) * sizeof(int), ctx->stream));
    CK(cudaMemsetAsync(ctx->uf.p, 0, (size_t)B * nn * 2 * (ctx->f64 ? 8 : 4), ctx->stream));
    int rc = alloc_sat(ctx, B);
    if (rc) return rc;
    rc = alloc_spans(ctx);
    if (rc) return rc;
    ctx->h_st.assign(B, Carto());
    ctx->params_set = false;
    ctx->ran = false;
    invalidate_graph(ctx);
    return DET_OK;
}

// Raster of the batch start vertices (pos_init) into labels/cnt_acc, growing the span
// capacity until no row overflows.  Leaves the counts in cnt_acc.
static int raster_start(det_ctx* ctx) {
    for (int attempt = 0; attempt < 8; ++attempt) {
        const long long nrow = (long long)ctx->B * ctx->n_rows;
        if (ctx->s64) {
            CK(cudaMemcpyAsync(ctx->pos0.p, ctx->pos_init.p, (size_t)nrow * sizeof(double2), cudaMemcpyDeviceToDevice,
                               ctx->stream));
        } else {  // float32 state: the start rows rounded once; the start raster stays on the exact rows
            k_rows_to_f32<<<(unsigned)std::min<long long>((nrow + 255) / 256, 4096), 256, 0, ctx->stream>>>(
                ctx->pos_init.p, nrow, reinterpret_cast<float2*>(ctx->pos0.p));
        }
        const Topo T = make_topo(ctx);
        const Bufs D = make_bufs(ctx);
        Bufs D0 = D;
        D0.pos0 = ctx->pos_init.p;
        k_init_state<<<(ctx->B + 127) / 128, 128, 0, ctx->stream>>>(D);
        CK(cudaMemsetAsync(ctx->cnt_acc.p, 0, (size_t)ctx->B * (ctx->R + 1) * sizeof(int), ctx->stream));
        launch_region(ctx, T, D0, M_RASTER, G_ALWAYS, 0, true);
        launch_row(ctx, T, D, G_ALWAYS, -1);
        CK(cudaGetLastError());
        std::vector<Carto> hs(ctx->B);
        std::vector<int> ms(ctx->B);
        CK(cudaMemcpyAsync(hs.data(), ctx->st.p, ctx->B * sizeof(Carto), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(ms.data(), ctx->maxspan.p, ctx->B * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        int mx = 0;
        bool ovf = false, tog = false;
        for (int b = 0; b < ctx->B; ++b) {
            mx = std::max(mx, ms[b]);
            ovf |= (hs[b].err & E_SPAN_OVF) != 0;
            tog |= (hs[b].err & E_TOGGLE_OVF) != 0;
        }
        if (tog) {  // > RW_TCAP crossings on one scanline of a region: redo with the bitmap raster
            if (ctx->bitmap_raster) return fail(ctx, DET_E_STATE, "toggle overflow in the bitmap raster");
            ctx->bitmap_raster = true;
            invalidate_graph(ctx);
            continue;
        }
        const int want = std::max(64, 2 * mx + 32);  // headroom for deformation
        if (!ovf) {
            if (ctx->cap < want) {
                ctx->cap = want;
                int rc = alloc_spans(ctx);
                if (rc) return rc;
            }
            return DET_OK;
        }
        ctx->cap = std::max(want, ctx->cap * 2);
        int rc = alloc_spans(ctx);
        if (rc) return rc;
    }
    return fail(ctx, DET_E_STATE, "span capacity did not converge");
}

// ================================ C-ABI ======================================
extern "C" {

static int labels_to_host(det_ctx* ctx, int b, int32_t* out);
static const double2* state_rows(det_ctx* ctx, int b);


int det_abi_version(void) { return 1; }

int det_debug_guard_check(long long* n_live, long long* n_bad) {
    if (!n_live || !n_bad) return DET_E_ARG;
    std::lock_guard<std::recursive_mutex> cap(g_guard_capture_mu);
    std::lock_guard<std::mutex> lk(g_guard_mu);
    long long bad = g_guard_bad_freed;
    for (const GuardAlloc& g : g_guard_live) bad += guard_intact(g) ? 0 : 1;
    *n_live = (long long)g_guard_live.size();
    *n_bad = bad;
    return guard_mode() ? DET_OK : DET_E_STATE;
}

int det_host_alloc(size_t bytes, void** out) {
    if (!out) return DET_E_ARG;
    *out = nullptr;
    if (bytes == 0) return DET_OK;
    return cudaHostAlloc(out, bytes, cudaHostAllocDefault) == cudaSuccess ? DET_OK : DET_E_CUDA;
}

int det_host_free(void* p) {
    if (!p) return DET_OK;
    return cudaFreeHost(p) == cudaSuccess ? DET_OK : DET_E_CUDA;
}

// Synchronous copies on the context's own stream (never the legacy default stream, which a
// cudaStreamNonBlocking context stream does not order against).
static cudaError_t copy_sync(det_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream);
    return e != cudaSuccess ? e : cudaStreamSynchronize(ctx->stream);
}

const char* det_last_error(const det_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int det_device_info(int device, char* buf, int buflen) {
    cudaDeviceProp p;
    cudaError_t e = cudaGetDeviceProperties(&p, device);
    if (e != cudaSuccess) {
        snprintf(buf, buflen, "cuda error: %s", cudaGetErrorString(e));
        return DET_E_CUDA;
    }
    snprintf(buf, buflen, "%s sm_%d%d SMs=%d L2=%dB smem/block=%zu", p.name, p.major, p.minor, p.multiProcessorCount,
             p.l2CacheSize, p.sharedMemPerBlockOptin);
    return DET_OK;
}

int det_ctx_create(int device, int k, int precision, det_ctx** out) {
    if (!out) return DET_E_ARG;
    *out = nullptr;
    if (k < 4 || k > 13 || precision < DET_PREC_FLOAT32 || precision > DET_PREC_MIXED) return DET_E_ARG;
    det_ctx* ctx = new det_ctx();
    if (const char* e = getenv("DET_SEP_CTRL")) ctx->sep_ctrl = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_SPLIT_ADVECT")) ctx->split_adv = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_RASTER_RO")) ctx->raster_ro = atoi(e) != 0;    // A/B switch (diagnostics)
    if (const char* e = getenv("DET_UNIQ_ADVECT")) ctx->uniq_adv = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_SAT1W")) ctx->sat1w = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_SAT3W")) ctx->sat3w = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_SAT3X")) ctx->sat3x = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_UQ_STATE")) ctx->uq_state = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_FUSE_ADVECT")) ctx->fuse_adv = atoi(e) != 0;  // A/B switch (diagnostics)
    if (const char* e = getenv("DET_SAT1X")) ctx->sat1x = atoi(e) != 0;  // A/B switch (diagnostics)
    ctx->device = device;
    ctx->k = k;
    ctx->n = 1 << k;
    ctx->f64 = precision == DET_PREC_FLOAT64;
    ctx->s64 = precision != DET_PREC_FLOAT32;
    ctx->H = std::min(8, ctx->n);
    ctx->nb = ctx->n / ctx->H;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        int rc = DET_E_CUDA;
        delete ctx;
        return rc;
    }
    *out = ctx;
    return DET_OK;
}

void det_ctx_destroy(det_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    invalidate_graph(ctx);
    for (cudaStream_t s : ctx->gstreams) cudaStreamDestroy(s);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int det_set_groups(det_ctx* ctx, int groups) {
    if (!ctx || groups < 1 || groups > 16) return fail(ctx, DET_E_ARG, "groups must be in [1, 16]");
    ctx->groups = groups;
    invalidate_graph(ctx);
    return DET_OK;
}

int det_set_band_height(det_ctx* ctx, int h) {
    if (!ctx || h < 0 || (h & (h - 1)) || h > ctx->n)
        return fail(ctx, DET_E_ARG, "band height must be a power of two <= n (0: automatic)");
    cudaSetDevice(ctx->device);
    ctx->h_fixed = h != 0;
    ctx->H = h ? h : auto_band_height(ctx->n, std::max(ctx->B, 1));
    ctx->nb = ctx->n / ctx->H;
    invalidate_graph(ctx);
    if (ctx->B > 0) return alloc_sat(ctx, ctx->B);
    return DET_OK;
}

int det_load_map(det_ctx* ctx, const double* xy, int n_rows, const int32_t* ring_start, int n_rings,
                 const int32_t* ring_region, const int32_t* region_rank, int n_regions) {
    if (!ctx || !xy || !ring_start || !ring_region || !region_rank || n_rows <= 0 || n_rings <= 0 || n_regions <= 0)
        return fail(ctx, DET_E_ARG, "invalid map arguments");
    cudaSetDevice(ctx->device);
    if (ring_start[0] != 0 || ring_start[n_rings] != n_rows) return fail(ctx, DET_E_ARG, "ring_start must span all rows");
    std::vector<int> reg_row0(n_regions + 1, -1), reg_ring0(n_regions + 1, 0), rank_reg(n_regions, -1);
    int prev_region = -1;
    for (int q = 0; q < n_rings; ++q) {
        const int r = ring_region[q];
        if (r < 0 || r >= n_regions || r < prev_region) return fail(ctx, DET_E_ARG, "rings must be grouped by region in order");
        if (ring_start[q + 1] - ring_start[q] < 1) return fail(ctx, DET_E_ARG, "empty ring");
        while (prev_region < r) {
            ++prev_region;
            reg_row0[prev_region] = ring_start[q];
            reg_ring0[prev_region] = q;
        }
    }
    if (prev_region != n_regions - 1) return fail(ctx, DET_E_ARG, "every region needs at least one ring");
    reg_row0[n_regions] = n_rows;
    reg_ring0[n_regions] = n_rings;
    for (int r = 0; r < n_regions; ++r) {
        const int k = region_rank[r];
        if (k < 0 || k >= n_regions || rank_reg[k] != -1) return fail(ctx, DET_E_ARG, "region_rank must be a permutation");
        rank_reg[k] = r;
    }
    // vertex rows are stored per ring row (coalesced); rows duplicating a shared vertex
    // evolve bit-identically, so no de-duplication is needed
    ctx->R = n_regions;
    ctx->n_rows = n_rows;
    ctx->n_rings = n_rings;
    CK(ctx->xy_rows.alloc(n_rows));
    CK(cudaMemcpyAsync(ctx->xy_rows.p, xy, (size_t)n_rows * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    ctx->h_ring_start.assign(ring_start, ring_start + n_rings + 1);
    ctx->h_region_ring0 = reg_ring0;
    CK(ctx->region_row0.alloc(n_regions + 1));
    CK(ctx->region_ring0.alloc(n_regions + 1));
    CK(ctx->ring_start.alloc(n_rings + 1));
    CK(ctx->region_rank.alloc(n_regions));
    CK(ctx->rank_region.alloc(n_regions));
    CK(copy_sync(ctx, ctx->region_row0.p, reg_row0.data(), (n_regions + 1) * sizeof(int), cudaMemcpyHostToDevice));
    CK(copy_sync(ctx, ctx->region_ring0.p, reg_ring0.data(), (n_regions + 1) * sizeof(int), cudaMemcpyHostToDevice));
    CK(copy_sync(ctx, ctx->ring_start.p, ring_start, (n_rings + 1) * sizeof(int), cudaMemcpyHostToDevice));
    CK(copy_sync(ctx, ctx->region_rank.p, region_rank, n_regions * sizeof(int), cudaMemcpyHostToDevice));
    CK(copy_sync(ctx, ctx->rank_region.p, rank_reg.data(), n_regions * sizeof(int), cudaMemcpyHostToDevice));
    // unique vertices: rows with bit-identical coordinates, numbered by first occurrence (so the
    // representative rows ascend: near-coalesced reads).  Open-addressing hash on the coordinate
    // bits; a re-load of the same rows (the public API re-uploads a map per call) reuses the result.
    const bool same_rows = (int)ctx->h_xy_prev.size() == 2 * n_rows &&
                           !memcmp(ctx->h_xy_prev.data(), xy, (size_t)n_rows * 2 * sizeof(double));
    if (!same_rows) {
        ctx->h_xy_prev.assign(xy, xy + (size_t)2 * n_rows);
        const uint64_t* bits = reinterpret_cast<const uint64_t*>(xy);
        size_t cap = 1;
        while (cap < (size_t)2 * n_rows) cap <<= 1;
        std::vector<int> slot(cap, -1);  // representative row of each occupied slot
        std::vector<int> uid(n_rows), row0;
        int U = 0;
        for (int v = 0; v < n_rows; ++v) {
            const uint64_t hx = bits[2 * v], hy = bits[2 * v + 1];
            size_t h = (size_t)((hx * 0x9E3779B97F4A7C15ull) ^ (hy + 0x632BE59BD9B4E019ull + (hx << 6) + (hx >> 2)));
            h ^= h >> 29;
            for (size_t i = h & (cap - 1);; i = (i + 1) & (cap - 1)) {
                const int r = slot[i];
                if (r < 0) {
                    slot[i] = v;
                    uid[v] = U++;
                    row0.push_back(v);
                    break;
                }
                if (bits[2 * r] == hx && bits[2 * r + 1] == hy) {
                    uid[v] = uid[r];
                    break;
                }
            }
        }
        std::vector<int> off(U + 1, 0), rows(n_rows);
        for (int v = 0; v < n_rows; ++v) ++off[uid[v] + 1];
        for (int u = 0; u < U; ++u) off[u + 1] += off[u];
        std::vector<int> cur(off.begin(), off.end() - 1);
        for (int v = 0; v < n_rows; ++v) rows[cur[uid[v]]++] = v;
        ctx->n_uniq = U;
        ctx->h_uq_off = off;
        ctx->h_uq_rows = rows;
        ctx->h_uq_row0 = row0;
        ctx->h_row_uniq = uid;
    }
    if (!same_rows) {  // (unchanged rows: the device tables still hold this map's)
        const int U = ctx->n_uniq;
        const std::vector<int>& off = ctx->h_uq_off;
        const std::vector<int>& rows = ctx->h_uq_rows;
        const std::vector<int>& row0 = ctx->h_uq_row0;
        CK(ctx->uq_row0.alloc(U));
        CK(ctx->uq_off.alloc(U + 1));
        CK(ctx->uq_rows.alloc(n_rows));
        CK(copy_sync(ctx, ctx->uq_row0.p, row0.data(), (size_t)U * sizeof(int), cudaMemcpyHostToDevice));
        CK(copy_sync(ctx, ctx->uq_off.p, off.data(), (size_t)(U + 1) * sizeof(int), cudaMemcpyHostToDevice));
        CK(copy_sync(ctx, ctx->uq_rows.p, rows.data(), (size_t)n_rows * sizeof(int), cudaMemcpyHostToDevice));
        CK(ctx->row_uniq.alloc(n_rows));
        CK(copy_sync(ctx, ctx->row_uniq.p, ctx->h_row_uniq.data(), (size_t)n_rows * sizeof(int), cudaMemcpyHostToDevice));
    }
    ctx->ua_ok = false;
    {  // ring successor of every row: O(1) for regions with many rings (holes, islands)
        std::vector<int> nxt(n_rows);
        for (int q = 0; q < n_rings; ++q)
            for (int v = ring_start[q]; v < ring_start[q + 1]; ++v) nxt[v] = v + 1 < ring_start[q + 1] ? v + 1 : ring_start[q];
        CK(ctx->row_next.alloc(n_rows));
        CK(copy_sync(ctx, ctx->row_next.p, nxt.data(), (size_t)n_rows * sizeof(int), cudaMemcpyHostToDevice));
    }
    ctx->B = 0;
    ctx->params_set = false;
    return DET_OK;
}

int det_set_batch(det_ctx* ctx, int batch, const double* xy, const double* stats) {
    if (!ctx || batch <= 0 || !stats) return fail(ctx, DET_E_ARG, "invalid batch arguments");
    if (ctx->n_rows == 0) return fail(ctx, DET_E_STATE, "det_load_map first");
    cudaSetDevice(ctx->device);
    if (batch != ctx->B) {
        int rc = alloc_batch(ctx, batch);
        if (rc) return rc;
    }
    const size_t rowb = (size_t)ctx->n_rows * sizeof(double2);
    // the unique-vertex advect needs every frame's start rows to keep the map's shared vertices
    // bit-identical (the loaded rows do; caller-given rows are checked)
    ctx->ua_ok = true;
    if (xy) {
        const uint64_t* bits = reinterpret_cast<const uint64_t*>(xy);
        for (int b = 0; b < batch && ctx->ua_ok; ++b) {
            const uint64_t* fb = bits + (size_t)b * ctx->n_rows * 2;
            for (int u = 0; u < ctx->n_uniq && ctx->ua_ok; ++u) {
                const int o0 = ctx->h_uq_off[u], o1 = ctx->h_uq_off[u + 1];
                const int r0 = ctx->h_uq_rows[o0];
                for (int i = o0 + 1; i < o1; ++i) {
                    const int v = ctx->h_uq_rows[i];
                    if (fb[2 * v] != fb[2 * r0] || fb[2 * v + 1] != fb[2 * r0 + 1]) { ctx->ua_ok = false; break; }
                }
            }
        }
    }
    if (xy) {
        CK(cudaMemcpyAsync(ctx->pos_init.p, xy, (size_t)batch * rowb, cudaMemcpyHostToDevice, ctx->stream));
    } else {  // one upload of the loaded rows, replicated on the device
        CK(cudaMemcpyAsync(ctx->pos_init.p, ctx->xy_rows.p, rowb, cudaMemcpyDeviceToDevice, ctx->stream));
        for (int b = 1; b < batch; ++b)
            CK(cudaMemcpyAsync(ctx->pos_init.p + (size_t)b * ctx->n_rows, ctx->pos_init.p, rowb, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    }
    CK(cudaMemcpyAsync(ctx->stats.p, stats, (size_t)batch * ctx->R * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->ran = false;
    return DET_OK;
}

int det_rasterize(det_ctx* ctx, int b, int32_t* labels_out, int64_t* counts_out) {
    if (!ctx || ctx->B == 0) return fail(ctx, DET_E_STATE, "det_set_batch first");
    if (b < 0 || b >= ctx->B) return fail(ctx, DET_E_ARG, "cartogram index out of range");
    cudaSetDevice(ctx->device);
    int rc = raster_start(ctx);
    if (rc) return rc;
    Carto hs;
    CK(copy_sync(ctx, &hs, ctx->st.p + b, sizeof(Carto), cudaMemcpyDeviceToHost));
    if (hs.err & E_NEGIDX) return fail(ctx, DET_E_VALUE, "'list' argument must have no negative elements");
    if (labels_out) {
        const int rc2 = labels_to_host(ctx, b, labels_out);
        if (rc2) return rc2;
    }
    if (counts_out) {
        std::vector<int> c(ctx->R + 1);
        CK(copy_sync(ctx, c.data(), ctx->cnt_acc.p + (size_t)b * (ctx->R + 1), (ctx->R + 1) * sizeof(int), cudaMemcpyDeviceToHost));
        for (int r = 0; r <= ctx->R; ++r) counts_out[r] = c[r];
    }
    CK(cudaMemsetAsync(ctx->cnt_acc.p, 0, (size_t)ctx->B * (ctx->R + 1) * sizeof(int), ctx->stream));
    ctx->ran = false;
    return DET_OK;
}

int det_set_params(det_ctx* ctx, const det_params* params, const double* weights_px) {
    if (!ctx || ctx->B == 0 || !params || !weights_px) return fail(ctx, DET_E_ARG, "invalid params");
    cudaSetDevice(ctx->device);
    ctx->h_prm.resize(ctx->B);
    for (int b = 0; b < ctx->B; ++b) {
        Params& p = ctx->h_prm[b];
        memset(&p, 0, sizeof(p));
        p.background_mass = params[b].background_mass;
        p.mult = params[b].bdv_multiplier;
        p.mean_density0 = params[b].mean_density0;
        p.S = params[b].total_statistic;
        p.mode = params[b].bdv_mode;
    }
    CK(cudaMemcpyAsync(ctx->weights.p, weights_px, (size_t)ctx->B * ctx->R * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->params_set = true;
    return DET_OK;
}

// *overflow: bit 0 = a row's spans overflowed the span buffer (grow and redo), bit 1 = a scanline
// overflowed k_region's toggle window (redo with the bitmap raster)
static int run_once(det_ctx* ctx, const det_criteria* crit, int* overflow) {
    *overflow = 0;
    const int B = ctx->B;
    const int tc = crit->max_iterations + 1;
    if (tc > ctx->trace_cap || ctx->trace.n < (size_t)B * ctx->trace_cap * 4) {
        ctx->trace_cap = std::max(std::max(tc, ctx->trace_cap), 1024);
        CK(ctx->trace.alloc((size_t)B * ctx->trace_cap * 4));
        invalidate_graph(ctx);
    }
    for (int b = 0; b < B; ++b) {
        ctx->h_prm[b].thr = crit->error_threshold;
        ctx->h_prm[b].window = crit->stagnation_window;
        ctx->h_prm[b].max_iter = crit->max_iterations;
    }
    CK(cudaMemcpyAsync(ctx->prm.p, ctx->h_prm.data(), B * sizeof(Params), cudaMemcpyHostToDevice, ctx->stream));
    int rc = raster_start(ctx);  // state 0 labels/counts (+ span capacity sizing)
    if (rc) return rc;
    {
        Carto hs;
        for (int b = 0; b < B; ++b) {
            CK(copy_sync(ctx, &hs, ctx->st.p + b, sizeof(Carto), cudaMemcpyDeviceToHost));
            if (hs.err & E_NEGIDX) return fail(ctx, DET_E_VALUE, "'list' argument must have no negative elements");
        }
    }
    rc = ensure_graph(ctx);
    if (rc) return rc;
    {
        const Topo T = make_topo(ctx);
        const Bufs D = make_bufs(ctx);
        k_ctrl<<<B, CTRL_THREADS, 0, ctx->stream>>>(T, D, 0, G_ACTIVE);
        CK(cudaGetLastError());
    }
    const int max_launches = crit->max_iterations / kGraphIters + 2;
    for (int l = 0; l < max_launches; ++l) {
        CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
        CK(cudaMemcpyAsync(ctx->h_st.data(), ctx->st.p, B * sizeof(Carto), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        bool any = false;
        for (int b = 0; b < B; ++b) {
            if (ctx->h_st[b].err & (E_SPAN_OVF | E_TOGGLE_OVF)) {
                for (int q = 0; q < B; ++q)
                    *overflow |= ((ctx->h_st[q].err & E_SPAN_OVF) ? 1 : 0) | ((ctx->h_st[q].err & E_TOGGLE_OVF) ? 2 : 0);
                return DET_OK;
            }
            any |= ctx->h_st[b].active != 0;
        }
        if (!any) break;
    }
    bool fin = false;
    for (int b = 0; b < B; ++b) fin |= ctx->h_st[b].final_pending != 0;
    if (fin) {
        const Topo T = make_topo(ctx);
        const Bufs D = make_bufs(ctx);
        launch_region(ctx, T, D, M_RASTER, G_FINAL, 2);
        launch_row(ctx, T, D, G_FINAL, 1);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(ctx->h_st.data(), ctx->st.p, B * sizeof(Carto), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int b = 0; b < B; ++b)
        *overflow |= ((ctx->h_st[b].err & E_SPAN_OVF) ? 1 : 0) | ((ctx->h_st[b].err & E_TOGGLE_OVF) ? 2 : 0);
    return DET_OK;
}

int det_run(det_ctx* ctx, const det_criteria* crit) {
    if (!ctx || !crit) return DET_E_ARG;
    if (!ctx->params_set) return fail(ctx, DET_E_STATE, "det_set_params first");
    if (crit->max_iterations <= 0 || crit->stagnation_window <= 0 || !(crit->error_threshold > 0))
        return fail(ctx, DET_E_ARG, "stopping criteria must all be positive");
    cudaSetDevice(ctx->device);
    for (int attempt = 0; attempt < 6; ++attempt) {
        int ovf = 0;
        ctx->bench_mode = false;
        int rc = run_once(ctx, crit, &ovf);
        if (rc) return rc;
        if (!ovf) {
            ctx->ran = true;
            return DET_OK;
        }
        if (ovf & 2) {  // a scanline collected more crossings than k_region's window: bitmap raster
            if (ctx->bitmap_raster) return fail(ctx, DET_E_STATE, "toggle overflow in the bitmap raster");
            ctx->bitmap_raster = true;
            invalidate_graph(ctx);
        }
        if (ovf & 1) {
            ctx->cap *= 2;  // a row collected more spans than the buffer holds: grow and redo
            rc = alloc_spans(ctx);
            if (rc) return rc;
        } else {
            CK(cudaMemsetAsync(ctx->rowcnt.p, 0, (size_t)ctx->B * ctx->n * sizeof(int), ctx->stream));
        }
    }
    return fail(ctx, DET_E_STATE, "span capacity did not converge");
}

// Cumulative time-step chain (temporal.py:162-246 with cumulative=True), device resident:
// frame t starts from frame t-1's deformed vertices without leaving the GPU.  Per frame the
// engine constants (engine.py:122-139) are derived from the frame's initial raster with the
// reference's float64 expressions; S[t] is the statistic total as the caller computed it.
int det_run_chain(det_ctx* ctx, int T, const double* stats, const double* S, const double* masses,
                  const det_criteria* crit, double* xy_out, det_result* res_out, int64_t* counts_out,
                  double* trace_out) {
    if (!ctx || T <= 0 || !stats || !S || !masses || !crit || !xy_out || !res_out || !counts_out || !trace_out)
        return fail(ctx, DET_E_ARG, "bad arguments");
    if (ctx->B != 1) return fail(ctx, DET_E_STATE, "det_set_batch(ctx, 1, ...) first");
    cudaSetDevice(ctx->device);
    const int R = ctx->R, nr = ctx->n_rows;
    const double m = (double)ctx->n * ctx->n;
    const int tstride = (crit->max_iterations + 1) * 4;
    std::vector<int> c0(R + 1);
    std::vector<double> w(R);
    for (int t = 0; t < T; ++t) {
        const double* s = stats + (size_t)t * R;
        det_result& res = res_out[t];
        memset(&res, 0, sizeof(res));
        res.collapsed_region = -1;
        CK(cudaMemcpyAsync(ctx->stats.p, s, R * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        int rc = raster_start(ctx);  // frame start raster (engine.py:128, check_collapse=True)
        if (rc) return rc;
        Carto hs;
        CK(copy_sync(ctx, &hs, ctx->st.p, sizeof(Carto), cudaMemcpyDeviceToHost));
        CK(copy_sync(ctx, c0.data(), ctx->cnt_acc.p, (R + 1) * sizeof(int), cudaMemcpyDeviceToHost));
        for (int r = 0; r <= R; ++r) counts_out[(size_t)t * (R + 1) + r] = c0[r];
        if (hs.err & E_NEGIDX) {
            res.status = DET_E_VALUE;
            res.stop_reason = DET_STOP_NEGINDEX;
            continue;
        }
        bool empty = false;
        for (int r = 0; r < R; ++r) empty |= c0[r] == 0;
        if (empty) {  // RasterizationError at engine construction: frame fails, chain keeps its geometry
            res.status = DET_E_RASTER;
            continue;
        }
        const double total_mass = S[t] + masses[t];
        for (int r = 0; r < R; ++r) w[r] = s[r] / total_mass * m;  // engine.py:138-139
        const double map0 = m - (double)c0[R];
        det_params p;
        memset(&p, 0, sizeof(p));
        p.background_mass = masses[t];
        p.bdv_multiplier = 1.0;  // temporal.py:190-196 leaves the engine's multiplier at its default
        p.mean_density0 = S[t] / map0;
        p.total_statistic = S[t];
        p.bdv_mode = DET_BDV_FIXED_MASS;
        rc = det_set_params(ctx, &p, w.data());
        if (rc) return rc;
        rc = det_run(ctx, crit);
        if (rc) return rc;
        rc = det_get_result(ctx, 0, &res);
        if (rc) return rc;
        if (res.stop_reason == DET_STOP_COLLAPSED || res.stop_reason == DET_STOP_BDV ||
            res.stop_reason == DET_STOP_NEGINDEX)
            continue;  // the frame failed; the next frame starts from the same geometry
        rc = det_get_counts(ctx, 0, counts_out + (size_t)t * (R + 1));
        if (rc) return rc;
        if (res.trace_len > 0) {
            rc = det_get_trace(ctx, 0, trace_out + (size_t)t * tstride);
            if (rc) return rc;
        }
        const double2* rows = state_rows(ctx, 0);
        CK(cudaMemcpyAsync(xy_out + (size_t)t * nr * 2, rows, nr * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(ctx->pos_init.p, rows, nr * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    ctx->ran = false;  // per-frame results were returned; the context now holds the chain's last start
    return DET_OK;
}

int det_bench_iterations(det_ctx* ctx, int iters) {
    if (!ctx || !ctx->ran || !ctx->params_set) return fail(ctx, DET_E_STATE, "det_run first");
    cudaSetDevice(ctx->device);
    if (!ctx->bench_mode) {
        // never-stopping criteria; every cartogram continues from its current state
        for (int b = 0; b < ctx->B; ++b) {
            ctx->h_prm[b].thr = 0.0;
            ctx->h_prm[b].window = 0x3fffffff;
            ctx->h_prm[b].max_iter = 0x3fffffff;
        }
        CK(cudaMemcpyAsync(ctx->prm.p, ctx->h_prm.data(), ctx->B * sizeof(Params), cudaMemcpyHostToDevice, ctx->stream));
        k_reactivate<<<(ctx->B + 127) / 128, 128, 0, ctx->stream>>>(make_bufs(ctx));
        CK(cudaGetLastError());
        int rc = ensure_graph(ctx);
        if (rc) return rc;
        ctx->bench_mode = true;
    }
    int done = 0;
    for (; done + kGraphIters <= iters; done += kGraphIters) CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
    // the remainder runs eagerly over the whole batch, on the unique-vertex state like the graph
    // (gathered in its first iteration, expanded in its last)
    const int rem = iters - done;
    for (int i = 0; i < rem; ++i)
        enqueue_iteration(ctx, 0, -1, nullptr, uqs_on(ctx) ? (2 | (i == 0 ? 1 : 0) | (i == rem - 1 ? 4 : 0)) : 0);
    CK(cudaGetLastError());
    return DET_OK;
}

int det_bench_kernel_times(det_ctx* ctx, int iters, float* ms_out) {
    // Per-kernel device time of `iters` eagerly launched iterations, CUDA events on the
    // context stream: ms_out[0..5] = sat1, sat2, sat3 (fused here as one launch_sat), region, row, ctrl
    if (!ctx || !ms_out) return DET_E_ARG;
    int rc = det_bench_iterations(ctx, 0);
    if (rc) return rc;
    cudaEvent_t ev[5];
    for (int i = 0; i < 5; ++i) CK(cudaEventCreate(&ev[i]));
    for (int i = 0; i < 4; ++i) ms_out[i] = 0.f;
    // diagnostics: DET_KT_REGION_MODE=1 times k_region's advect phase alone (raster skipped),
    // =2 its raster alone (the rows are not advected)
    const char* km = getenv("DET_KT_REGION_MODE");
    const int region_mode = (km && km[0] == '1') ? M_ADVECT : (km && km[0] == '2') ? M_RASTER : (M_ADVECT | M_RASTER);
    // DET_KT_ROW_MODE=-1 times k_row without the evaluation / LUT part of the control step
    const char* rm = getenv("DET_KT_ROW_MODE");
    const int row_mode = (rm && rm[0] == '-') ? -1 : 0;
    const Topo T = make_topo(ctx);
    const Bufs D = make_bufs(ctx);
    SatSrc S;
    memset(&S, 0, sizeof(S));
    // the graph's own kernels: on the unique-vertex state when the graph runs on it (gathered before
    // and expanded after the timed iterations, as at the ends of a graph launch)
    const bool uqs = uqs_on(ctx) && region_mode == (M_ADVECT | M_RASTER);
    if (uqs)
        k_uq_gather<<<dim3(std::min((ctx->n_uniq + 255) / 256, 1024), ctx->B), 256, 0, ctx->stream>>>(T, D, G_ACTIVE, ctx->uq_row0.p);
    for (int it = 0; it < iters; ++it) {
        CK(cudaEventRecord(ev[0], ctx->stream));
        const int fa = (uqs && fa_on(ctx)) ? (it & 1) : -1;  // (an even iteration count leaves buffer 0 current)
        launch_sat(ctx, T, D, S, G_ACTIVE, SRC_LABELS, OUT_U, ctx->f64 != 0, ctx->B, fa);
        CK(cudaEventRecord(ev[1], ctx->stream));
        launch_advect_raster(ctx, T, D, G_ACTIVE, region_mode, uqs, fa);
        CK(cudaEventRecord(ev[2], ctx->stream));
        launch_row_ctrl(ctx, T, D, G_ACTIVE, row_mode);  // includes the control step
        CK(cudaEventRecord(ev[3], ctx->stream));
        CK(cudaEventRecord(ev[4], ctx->stream));
        CK(cudaEventSynchronize(ev[4]));
        for (int q = 0; q < 4; ++q) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, ev[q], ev[q + 1]));
            ms_out[q] += t;
        }
    }
    if (uqs) k_uq_expand<<<dim3(std::min((ctx->n_rows + 255) / 256, 1024), ctx->B), 256, 0, ctx->stream>>>(T, D);
    CK(cudaGetLastError());
    for (int i = 0; i < 5; ++i) cudaEventDestroy(ev[i]);
    return DET_OK;
}

int det_time_iterations(det_ctx* ctx, int iters, float* ms_out) {
    if (!ctx || !ms_out) return DET_E_ARG;
    cudaSetDevice(ctx->device);
    int rc = det_bench_iterations(ctx, 0);  // enter bench mode (criteria that never stop)
    if (rc) return rc;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaEventRecord(e0, ctx->stream));
    rc = det_bench_iterations(ctx, iters);
    if (rc) return rc;
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(ms_out, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return DET_OK;
}

int det_progress(det_ctx* ctx, int32_t* next_iter_out, int32_t* active_out) {
    if (!ctx || ctx->B == 0) return fail(ctx, DET_E_STATE, "no batch");
    cudaSetDevice(ctx->device);
    std::vector<Carto> hs(ctx->B);
    CK(cudaMemcpyAsync(hs.data(), ctx->st.p, ctx->B * sizeof(Carto), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int b = 0; b < ctx->B; ++b) {
        if (next_iter_out) next_iter_out[b] = hs[b].next_iter;
        if (active_out) active_out[b] = hs[b].active;
    }
    return DET_OK;
}

int det_sync(det_ctx* ctx) {
    if (!ctx) return DET_E_ARG;
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

int det_get_result(det_ctx* ctx, int b, det_result* out) {
    if (!ctx || !out || b < 0 || b >= ctx->B || !ctx->ran) return fail(ctx, DET_E_STATE, "no result");
    const Carto& c = ctx->h_st[b];
    memset(out, 0, sizeof(*out));
    out->stop_reason = c.stop;
    out->iteration = c.res_iter;
    out->best_iteration = c.best_iter;
    out->collapsed_region = c.stop == S_COLLAPSED ? c.collapsed : -1;
    out->clamp_events = (int64_t)c.clamps;
    out->epsilon = c.eps;
    out->xi = c.xi;
    out->bdv = c.bdv;
    out->trace_len = c.trace_len;
    out->status = c.stop == S_COLLAPSED ? DET_E_COLLAPSE : ((c.stop == S_BDV || c.stop == S_NEGINDEX) ? DET_E_VALUE : DET_OK);
    return DET_OK;
}

static int result_src(det_ctx* ctx, int b) {
    const Carto& c = ctx->h_st[b];
    if (c.stop == S_STAGNATION) return 2;
    return 0;  // the state rows are advected in place in pos0
}

// Device pointer to cartogram b's rows of the returned state (or the start rows before a run).
static const double2* state_rows(det_ctx* ctx, int b) {
    const size_t off = (size_t)b * ctx->n_rows;
    if (!ctx->ran) return ctx->pos_init.p + off;
    const int src = result_src(ctx, b);
    const double2* p = src == 2 ? ctx->best.p : ctx->pos0.p;
    if (ctx->s64) return p + off;
    // float32 state: widen cartogram b's rows into its slot of rows64 (stream-ordered)
    if (ctx->rows64.alloc((size_t)ctx->B * ctx->n_rows) != cudaSuccess) return nullptr;
    k_rows_to_f64<<<(unsigned)std::min<int>((ctx->n_rows + 255) / 256, 2048), 256, 0, ctx->stream>>>(
        reinterpret_cast<const float2*>(p) + off, ctx->n_rows, ctx->rows64.p + off);
    return ctx->rows64.p + off;
}

int det_get_vertices(det_ctx* ctx, int b, double* xy_out) {
    if (!ctx || !xy_out || b < 0 || b >= ctx->B) return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    CK(cudaMemcpyAsync(xy_out, state_rows(ctx, b), ctx->n_rows * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

static int labels_to_host(det_ctx* ctx, int b, int32_t* out) {
    const size_t nn = (size_t)ctx->n * ctx->n;
    DVec<int> tmp;
    CK(tmp.alloc(nn));
    k_rank_to_index<<<592, 256, 0, ctx->stream>>>(ctx->labels.p + b * nn, ctx->rank_region.p, nn, tmp.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp.p, nn * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

int det_get_labels(det_ctx* ctx, int b, int32_t* out) {
    if (!ctx || !out || b < 0 || b >= ctx->B) return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    return labels_to_host(ctx, b, out);
}

int det_get_counts(det_ctx* ctx, int b, int64_t* out) {
    if (!ctx || !out || b < 0 || b >= ctx->B || !ctx->ran) return fail(ctx, DET_E_STATE, "no result");
    cudaSetDevice(ctx->device);
    std::vector<int> c(ctx->R + 1);
    CK(copy_sync(ctx, c.data(), ctx->cnt_state.p + (size_t)b * (ctx->R + 1), (ctx->R + 1) * sizeof(int), cudaMemcpyDeviceToHost));
    for (int r = 0; r <= ctx->R; ++r) out[r] = c[r];
    return DET_OK;
}

int det_get_region_error(det_ctx* ctx, int b, double* out) {
    if (!ctx || !out || b < 0 || b >= ctx->B || !ctx->ran) return fail(ctx, DET_E_STATE, "no result");
    cudaSetDevice(ctx->device);
    CK(copy_sync(ctx, out, ctx->rerr.p + (size_t)b * ctx->R, ctx->R * sizeof(double), cudaMemcpyDeviceToHost));
    return DET_OK;
}

int det_get_trace(det_ctx* ctx, int b, double* out) {
    if (!ctx || !out || b < 0 || b >= ctx->B || !ctx->ran) return fail(ctx, DET_E_STATE, "no result");
    cudaSetDevice(ctx->device);
    const int len = ctx->h_st[b].trace_len;
    if (len > 0)
        CK(copy_sync(ctx, out, ctx->trace.p + (size_t)b * ctx->trace_cap * 4, (size_t)len * 4 * sizeof(double),
                      cudaMemcpyDeviceToHost));
    return DET_OK;
}

int det_get_results(det_ctx* ctx, double* xy_out, int64_t* counts_out, double* err_out, double* trace_out,
                    int trace_rows) {
    if (!ctx || !ctx->ran) return fail(ctx, DET_E_STATE, "no result");
    if (trace_out && trace_rows < 0) return fail(ctx, DET_E_ARG, "bad trace_rows");
    cudaSetDevice(ctx->device);
    const int B = ctx->B, R = ctx->R;
    cudaStream_t s = ctx->stream;
    if (xy_out) {
        bool all_state = !ctx->s64;  // float32 state, no frame returning its best rows: one widen, one copy
        for (int b = 0; b < B && all_state; ++b) all_state = result_src(ctx, b) == 0;
        if (all_state) {
            const long long len = (long long)B * ctx->n_rows;
            CK(ctx->rows64.alloc((size_t)len));
            k_rows_to_f64<<<(unsigned)std::min<long long>((len + 255) / 256, 8192), 256, 0, s>>>(
                reinterpret_cast<const float2*>(ctx->pos0.p), len, ctx->rows64.p);
            CK(cudaMemcpyAsync(xy_out, ctx->rows64.p, (size_t)len * sizeof(double2), cudaMemcpyDeviceToHost, s));
        } else {
            for (int b = 0; b < B; ++b)
                CK(cudaMemcpyAsync(xy_out + (size_t)b * ctx->n_rows * 2, state_rows(ctx, b),
                                   ctx->n_rows * sizeof(double2), cudaMemcpyDeviceToHost, s));
        }
    }
    std::vector<int> c;
    if (counts_out) {
        c.resize((size_t)B * (R + 1));
        CK(cudaMemcpyAsync(c.data(), ctx->cnt_state.p, c.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    if (err_out) CK(cudaMemcpyAsync(err_out, ctx->rerr.p, (size_t)B * R * sizeof(double), cudaMemcpyDeviceToHost, s));
    const int rows = std::min(trace_rows, ctx->trace_cap);
    if (trace_out && rows > 0)
        CK(cudaMemcpy2DAsync(trace_out, (size_t)trace_rows * 4 * sizeof(double), ctx->trace.p,
                             (size_t)ctx->trace_cap * 4 * sizeof(double), (size_t)rows * 4 * sizeof(double), B,
                             cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t i = 0; i < c.size(); ++i) counts_out[i] = c[i];
    return DET_OK;
}

int det_get_areas(det_ctx* ctx, int b, double* out) {
    if (!ctx || !out || b < 0 || b >= ctx->B) return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    DVec<double> tmp;
    CK(tmp.alloc(ctx->R));
    const Topo T = make_topo(ctx);
    k_areas<<<ctx->R, 128, 0, ctx->stream>>>(T, state_rows(ctx, b), ctx->ring_start.p, ctx->region_ring0.p, tmp.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp.p, ctx->R * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

static int field_impl(det_ctx* ctx, const double* d, double* u_out, double* channels_out, double* total_out,
                      bool full_mapping) {
    const size_t nn = (size_t)ctx->n * ctx->n;
    int rc = alloc_sat(ctx, std::max(ctx->B, 1));
    if (rc) return rc;
    CK(ctx->dense.alloc(nn));
    CK(ctx->uf64.alloc(nn * 2));
    if (channels_out) CK(ctx->ch8.alloc(nn * 8));
    CK(cudaMemcpyAsync(ctx->dense.p, d, nn * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    DVec<Carto> dummy;
    CK(dummy.alloc(1));
    CK(cudaMemsetAsync(dummy.p, 0, sizeof(Carto), ctx->stream));
    const Topo T = make_topo(ctx);
    Bufs D = make_bufs(ctx);
    D.B = 1;
    D.st = dummy.p;
    D.uf = ctx->uf64.p;
    SatSrc S;
    memset(&S, 0, sizeof(S));
    S.d = ctx->dense.p;
    S.scale = 1.0;
    S.offset = 0.0;
    S.ch8 = ctx->ch8.p;
    // pass 1: total mass C (and the 8 channels of d itself when requested)
    launch_sat(ctx, T, D, S, G_ALWAYS, SRC_DENSE, channels_out ? OUT_CH8 : OUT_U, true, 1);
    CK(cudaGetLastError());
    double C = 0.0;
    CK(cudaMemcpyAsync(&C, ctx->rowfull.p + ctx->n, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (total_out) *total_out = C;
    if (channels_out) CK(copy_sync(ctx, channels_out, ctx->ch8.p, nn * 8 * sizeof(double), cudaMemcpyDeviceToHost));
    if (u_out) {
        if (!(C > 0)) return fail(ctx, DET_E_NUMERIC, "mapping undefined for zero total density");
        if (full_mapping) {  // t(d) itself (displacement.py:102-131)
            S.scale = 1.0;
            S.offset = 0.0;
            S.outscale = 0.5 / C;
        } else {             // u = t(d) - t(const) via the residual density (displacement.py:198-206)
            S.scale = (double)nn / C;
            S.offset = -1.0;
            S.outscale = 0.0;
        }
        launch_sat(ctx, T, D, S, G_ALWAYS, SRC_DENSE, OUT_U, true, 1);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(u_out, ctx->uf64.p, nn * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return DET_OK;
}

int det_field(det_ctx* ctx, const double* d, double* u_out, double* channels_out, double* total_out) {
    if (!ctx || !d) return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    return field_impl(ctx, d, u_out, channels_out, total_out, false);
}

int det_mapping(det_ctx* ctx, const double* d, double* t_out) {
    if (!ctx || !d || !t_out) return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    return field_impl(ctx, d, t_out, nullptr, nullptr, true);
}

// mapping_grid / residual_field (displacement.py:102-131,198-206) from given channels
int det_mapping_channels(det_ctx* ctx, const double* channels, double total, const double* base, double* t_out) {
    if (!ctx || !channels || !t_out) return fail(ctx, DET_E_ARG, "bad arguments");
    if (!(total > 0)) return fail(ctx, DET_E_NUMERIC, "mapping undefined for zero total density");
    cudaSetDevice(ctx->device);
    const size_t nn = (size_t)ctx->n * ctx->n;
    DVec<double> ch, bs, out;
    CK(ch.alloc(nn * 8));
    CK(out.alloc(nn * 2));
    CK(cudaMemcpyAsync(ch.p, channels, nn * 8 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if (base) {
        CK(bs.alloc(nn * 2));
        CK(cudaMemcpyAsync(bs.p, base, nn * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    k_map_grid<<<(unsigned)std::min<size_t>((nn + 255) / 256, 148 * 16), 256, 0, ctx->stream>>>(
        ch.p, total, ctx->n, base ? bs.p : nullptr, out.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(t_out, out.p, nn * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

// mapping_point (displacement.py:150-170) at n_pts points from given channels
int det_mapping_points(det_ctx* ctx, const double* channels, double total, const double* xy, int n_pts,
                       double* out) {
    if (!ctx || !channels || !xy || !out || n_pts < 0) return fail(ctx, DET_E_ARG, "bad arguments");
    if (!(total > 0)) return fail(ctx, DET_E_NUMERIC, "mapping undefined for zero total density");
    cudaSetDevice(ctx->device);
    if (n_pts == 0) return DET_OK;
    const size_t nn = (size_t)ctx->n * ctx->n;
    DVec<double> ch, pin, pout;
    CK(ch.alloc(nn * 8));
    CK(pin.alloc((size_t)n_pts * 2));
    CK(pout.alloc((size_t)n_pts * 2));
    CK(cudaMemcpyAsync(ch.p, channels, nn * 8 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(pin.p, xy, (size_t)n_pts * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    k_map_points<<<(n_pts + 127) / 128, 128, 0, ctx->stream>>>(ch.p, total, ctx->n, (const double2*)pin.p, n_pts,
                                                              (double2*)pout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, pout.p, (size_t)n_pts * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

int det_density(det_ctx* ctx, const int32_t* labels, const double* stats, int n_regions, double bdv, double* d_out,
                int64_t* counts_out) {
    if (!ctx || !labels || !stats || n_regions <= 0) return fail(ctx, DET_E_ARG, "bad arguments");
    if (!(bdv > 0)) return fail(ctx, DET_E_VALUE, "bdv must be positive");
    cudaSetDevice(ctx->device);
    const size_t nn = (size_t)ctx->n * ctx->n;
    DVec<int> lab, cnt;
    DVec<double> st, d;
    CK(lab.alloc(nn));
    CK(cnt.alloc(n_regions + 1));
    CK(st.alloc(n_regions));
    CK(d.alloc(nn));
    CK(cudaMemcpyAsync(lab.p, labels, nn * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(st.p, stats, n_regions * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(cnt.p, 0, (n_regions + 1) * sizeof(int), ctx->stream));
    k_hist<<<592, 256, 0, ctx->stream>>>(lab.p, nn, n_regions, cnt.p);
    std::vector<int> hc(n_regions + 1);
    CK(cudaMemcpyAsync(hc.data(), cnt.p, (n_regions + 1) * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < n_regions; ++r)
        if (hc[r] == 0) return fail(ctx, DET_E_RASTER, "cannot build density with zero-pixel regions");
    if (counts_out)
        for (int r = 0; r <= n_regions; ++r) counts_out[r] = hc[r];
    if (d_out) {
        k_density<<<592, 256, 0, ctx->stream>>>(lab.p, nn, n_regions, st.p, cnt.p, bdv, d.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(d_out, d.p, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return DET_OK;
}

int det_interpolate(det_ctx* ctx, const double* a, const double* b, long long len, const double* fracs, int n_frac,
                    double* out) {
    if (!ctx || !a || !b || !fracs || !out || len < 0 || n_frac < 0) return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    if (len == 0 || n_frac == 0) return DET_OK;
    DVec<double> da, db, df, dout;
    CK(da.alloc(len));
    CK(db.alloc(len));
    CK(df.alloc(n_frac));
    CK(dout.alloc((size_t)len * n_frac));
    CK(cudaMemcpyAsync(da.p, a, len * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(db.p, b, len * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(df.p, fracs, n_frac * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    k_interpolate<<<592, 256, 0, ctx->stream>>>(da.p, db.p, len, df.p, n_frac, dout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout.p, (size_t)len * n_frac * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

int det_advect(det_ctx* ctx, const double* u, const double* xy, int n_pts, double* xy_out, int64_t* clamps) {
    if (!ctx || !u || !xy || !xy_out || n_pts < 0) return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    const size_t nn = (size_t)ctx->n * ctx->n;
    CK(ctx->uf64.alloc(nn * 2));
    CK(ctx->pts_in.alloc((size_t)n_pts * 2));
    CK(ctx->pts_out.alloc((size_t)n_pts * 2));
    CK(ctx->clampbuf.alloc(1));
    CK(cudaMemcpyAsync(ctx->uf64.p, u, nn * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->pts_in.p, xy, (size_t)n_pts * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->clampbuf.p, 0, sizeof(unsigned long long), ctx->stream));
    if (n_pts > 0)
        k_advect_points<<<(n_pts + 255) / 256, 256, 0, ctx->stream>>>(ctx->uf64.p, ctx->n, (const double2*)ctx->pts_in.p,
                                                                      n_pts, (double2*)ctx->pts_out.p, ctx->clampbuf.p);
    CK(cudaGetLastError());
    unsigned long long c = 0;
    CK(cudaMemcpyAsync(xy_out, ctx->pts_out.p, (size_t)n_pts * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&c, ctx->clampbuf.p, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (clamps) *clamps = (int64_t)c;
    return DET_OK;
}


// ---------------- frame quality metrics (metrics.py:82-162, geomodel.py:380-415) ----------------

static int upload_layout(det_ctx* ctx, const double* xy, int n_rows, int frames, const int32_t* ring_start,
                         int n_rings, const int32_t* ring_region, int n_regions, DVec<double2>& dxy,
                         DVec<int>& drs, DVec<int>& drr0) {
    if (!xy || !ring_start || !ring_region || n_rows <= 0 || n_rings <= 0)
        return fail(ctx, DET_E_ARG, "invalid map layout");
    if (ring_start[0] != 0 || ring_start[n_rings] != n_rows) return fail(ctx, DET_E_ARG, "ring_start must span all rows");
    std::vector<int> r0(n_regions + 1, 0);
    int prev = -1;
    for (int q = 0; q < n_rings; ++q) {
        const int r = ring_region[q];
        if (r < 0 || r >= n_regions || r < prev) return fail(ctx, DET_E_ARG, "rings must be grouped by region in order");
        if (ring_start[q + 1] - ring_start[q] < 1) return fail(ctx, DET_E_ARG, "empty ring");
        while (prev < r) r0[++prev] = q;
    }
    if (prev != n_regions - 1) return fail(ctx, DET_E_ARG, "every region needs at least one ring");
    r0[n_regions] = n_rings;
    CK(dxy.alloc((size_t)n_rows * frames));
    CK(drs.alloc(n_rings + 1));
    CK(drr0.alloc(n_regions + 1));
    CK(cudaMemcpyAsync(dxy.p, xy, (size_t)n_rows * frames * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(drs.p, ring_start, (n_rings + 1) * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(drr0.p, r0.data(), (n_regions + 1) * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // r0 is a host temporary
    return DET_OK;
}

int det_shape_metrics(det_ctx* ctx, int n_regions, const double* xy_a, int rows_a, const int32_t* ring_start_a,
                      int rings_a, const int32_t* ring_region_a, const double* xy_b, int rows_b,
                      const int32_t* ring_start_b, int rings_b, const int32_t* ring_region_b, int frames,
                      int raster_k, int rescale, double* hamming, double* area_b, double* cent_a, double* cent_b,
                      int32_t* status) {
    if (!ctx || n_regions <= 0 || frames <= 0 || !hamming || !area_b || !cent_a || !cent_b || !status)
        return fail(ctx, DET_E_ARG, "bad arguments");
    if (raster_k < 0 || raster_k > 8) return fail(ctx, DET_E_ARG, "raster_k must be in [0, 8]");
    cudaSetDevice(ctx->device);
    const size_t R = (size_t)n_regions, F = (size_t)frames;
    DVec<double2> da, db, dca, dcb;
    DVec<int> rsa, r0a, rsb, r0b, dst;
    DVec<double> dh, dar;
    int rc = upload_layout(ctx, xy_a, rows_a, 1, ring_start_a, rings_a, ring_region_a, n_regions, da, rsa, r0a);
    if (rc) return rc;
    rc = upload_layout(ctx, xy_b, rows_b, frames, ring_start_b, rings_b, ring_region_b, n_regions, db, rsb, r0b);
    if (rc) return rc;
    CK(dh.alloc(R * F));
    CK(dar.alloc(R * F));
    CK(dca.alloc(R));
    CK(dcb.alloc(R * F));
    CK(dst.alloc(R * F));
    const ShapeLayout La{da.p, rsa.p, r0a.p, rows_a}, Lb{db.p, rsb.p, r0b.p, rows_b};
    k_shape<<<dim3((unsigned)R, (unsigned)F), MK_THREADS, 0, ctx->stream>>>(La, Lb, n_regions, raster_k, rescale, dh.p,
                                                                            dar.p, dca.p, dcb.p, dst.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(hamming, dh.p, R * F * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(area_b, dar.p, R * F * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(cent_a, dca.p, R * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(cent_b, dcb.p, R * F * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(status, dst.p, R * F * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

int det_adjacency(det_ctx* ctx, const double* xy, int frames, int n_rows, const int32_t* row_region, int n_regions,
                  double epsilon, int32_t* pairs, long long cap, long long* n_pairs) {
    if (!ctx || !xy || !row_region || frames <= 0 || n_rows <= 0 || n_regions <= 0 || !n_pairs || cap < 0 ||
        (cap > 0 && !pairs))
        return fail(ctx, DET_E_ARG, "bad arguments");
    if (!(epsilon > 0.0)) return fail(ctx, DET_E_ARG, "epsilon must be positive");
    for (int v = 0; v < n_rows; ++v)
        if (row_region[v] < 0 || row_region[v] >= n_regions) return fail(ctx, DET_E_ARG, "row_region out of range");
    cudaSetDevice(ctx->device);
    const long long n = (long long)n_rows * frames;
    if (n >= (1LL << 31)) return fail(ctx, DET_E_ARG, "too many vertex rows in one adjacency batch");
    const int R_ = n_regions;
    cudaStream_t s = ctx->stream;
    DVec<double2> dxy;
    DVec<long long> cx, cy, mm;
    DVec<unsigned long long> keys, skeys, uk, pk, spk, rk, npair;
    DVec<int> nuk, rc, nrun, dreg;
    DVec<char> tmp;
    CK(dxy.alloc(n));
    CK(dreg.alloc(n_rows));
    CK(cx.alloc(n));
    CK(cy.alloc(n));
    CK(mm.alloc(4));
    CK(cudaMemcpyAsync(dxy.p, xy, (size_t)n * sizeof(double2), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dreg.p, row_region, (size_t)n_rows * sizeof(int), cudaMemcpyHostToDevice, s));
    const unsigned nb = (unsigned)((n + 255) / 256);
    k_adj_cells<<<nb, 256, 0, s>>>(dxy.p, n, epsilon, cx.p, cy.p);
    CK(cudaGetLastError());
    auto run_cub = [&](auto&& fn) -> cudaError_t {  // size query, then the call
        size_t bytes = 0;
        cudaError_t e = fn((void*)nullptr, bytes);
        if (e != cudaSuccess) return e;
        e = tmp.alloc(bytes);
        if (e != cudaSuccess) return e;
        return fn((void*)tmp.p, bytes);
    };
    const int ni = (int)n;
    CK(run_cub([&](void* t, size_t& b) { return cub::DeviceReduce::Min(t, b, cx.p, mm.p + 0, ni, s); }));
    CK(run_cub([&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, cx.p, mm.p + 1, ni, s); }));
    CK(run_cub([&](void* t, size_t& b) { return cub::DeviceReduce::Min(t, b, cy.p, mm.p + 2, ni, s); }));
    CK(run_cub([&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, cy.p, mm.p + 3, ni, s); }));
    long long h_mm[4];
    CK(cudaMemcpyAsync(h_mm, mm.p, sizeof(h_mm), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    AdjGrid g;
    g.mx = h_mm[0] - 1;
    g.my = h_mm[2] - 1;
    g.sx = h_mm[1] - h_mm[0] + 3;
    g.sy = h_mm[3] - h_mm[2] + 3;
    g.R = R_;
    g.n_rows = n_rows;
    const long double span = (long double)frames * (long double)g.sx * (long double)g.sy * (long double)R_;
    if (span >= 9.0e18L) return fail(ctx, DET_E_ARG, "vertex extent too large for the adjacency cell grid");
    const unsigned long long maxkey = (unsigned long long)span;
    int end_bit = 1;
    while (end_bit < 64 && (maxkey >> end_bit)) ++end_bit;
    CK(keys.alloc(n));
    CK(skeys.alloc(n));
    CK(uk.alloc(n));
    CK(nuk.alloc(1));
    k_adj_keys<<<nb, 256, 0, s>>>(cx.p, cy.p, dreg.p, n, g, keys.p);
    CK(cudaGetLastError());
    CK(run_cub([&](void* t, size_t& b) { return cub::DeviceRadixSort::SortKeys(t, b, keys.p, skeys.p, ni, 0, end_bit, s); }));
    CK(run_cub([&](void* t, size_t& b) { return cub::DeviceSelect::Unique(t, b, skeys.p, uk.p, nuk.p, ni, s); }));
    unsigned long long pcap = (unsigned long long)n * 2 + 1024, h_np = 0;
    CK(npair.alloc(1));
    for (int attempt = 0; attempt < 2; ++attempt) {
        CK(pk.alloc(pcap));
        CK(cudaMemsetAsync(npair.p, 0, sizeof(unsigned long long), s));
        k_adj_pairs<<<nb, 256, 0, s>>>(uk.p, nuk.p, g, pk.p, pcap, npair.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&h_np, npair.p, sizeof(h_np), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (h_np <= pcap) break;
        pcap = h_np;
    }
    const int np_ = (int)h_np;
    std::vector<unsigned long long> h_keys;
    std::vector<int> h_cnt;
    int h_runs = 0;
    if (np_ > 0) {
        CK(spk.alloc(np_));
        CK(rk.alloc(np_));
        CK(rc.alloc(np_));
        CK(nrun.alloc(1));
        int pbits = 1;
        const unsigned long long pmax = (unsigned long long)frames * R_ * (unsigned long long)R_;
        while (pbits < 64 && (pmax >> pbits)) ++pbits;
        CK(run_cub([&](void* t, size_t& b) { return cub::DeviceRadixSort::SortKeys(t, b, pk.p, spk.p, np_, 0, pbits, s); }));
        CK(run_cub([&](void* t, size_t& b) {
            return cub::DeviceRunLengthEncode::Encode(t, b, spk.p, rk.p, rc.p, nrun.p, np_, s);
        }));
        CK(cudaMemcpyAsync(&h_runs, nrun.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        h_keys.resize(h_runs);
        h_cnt.resize(h_runs);
        CK(cudaMemcpyAsync(h_keys.data(), rk.p, h_runs * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(h_cnt.data(), rc.p, h_runs * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    long long cnt = 0;
    const unsigned long long RR = (unsigned long long)R_;
    for (int i = 0; i < h_runs; ++i) {
        if (h_cnt[i] < 2) continue;  // one shared corner is not an adjacency (geomodel.py:411-414)
        if (cnt < cap) {
            const unsigned long long k = h_keys[i];
            pairs[3 * cnt] = (int32_t)(k / (RR * RR));
            pairs[3 * cnt + 1] = (int32_t)((k / RR) % RR);
            pairs[3 * cnt + 2] = (int32_t)(k % RR);
        }
        ++cnt;
    }
    *n_pairs = cnt;
    return DET_OK;
}

int det_position_error(det_ctx* ctx, const double* cent_m, const double* cent_c, int frames, int n_regions,
                       double* sums_out, long long* degenerate_out) {
    if (!ctx || !cent_m || !cent_c || frames <= 0 || n_regions < 2 || !sums_out || !degenerate_out)
        return fail(ctx, DET_E_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    const size_t R = (size_t)n_regions, F = (size_t)frames;
    DVec<double2> bm, bc;
    DVec<double> part, out;
    DVec<long long> dg, dout;
    CK(bm.alloc(R));
    CK(bc.alloc(R * F));
    CK(part.alloc(R * F));
    CK(dg.alloc(R * F));
    CK(out.alloc(F));
    CK(dout.alloc(F));
    CK(cudaMemcpyAsync(bm.p, cent_m, R * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(bc.p, cent_c, R * F * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    k_poserr<<<dim3((unsigned)R, (unsigned)F), 128, 0, ctx->stream>>>(bm.p, bc.p, n_regions, part.p, dg.p);
    CK(cudaGetLastError());
    k_poserr_final<<<(unsigned)F, 256, 0, ctx->stream>>>(part.p, dg.p, n_regions, out.p, dout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(sums_out, out.p, F * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(degenerate_out, dout.p, F * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DET_OK;
}

}  // extern "C"
