// Shared device-side types and helpers of the DET engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace det {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t SENT = 0xffffffffu;
constexpr int REG_THREADS = 128;   // k_region block
constexpr int ROW_THREADS = 256;   // k_row block
constexpr int CTRL_THREADS = 1024;  // k_ctrl block (one per cartogram)
constexpr int CTRL_SEPARATE = -2;  // k_row ctrl_mode: leave the control step to k_ctrl

// M_POSTADV: raster the rows k_advect_rows just wrote (the advect runs as its own kernel)
enum Mode { M_ADVECT = 1, M_RASTER = 2, M_POSTADV = 4 };
enum Gate { G_ALWAYS = 0, G_ACTIVE = 1, G_FINAL = 2 };
enum Stop { S_RUNNING = 0, S_CONVERGED = 1, S_STAGNATION = 2, S_MAXITER = 3, S_COLLAPSED = 4, S_BDV = 5, S_NEGINDEX = 6 };
enum Err { E_SPAN_OVF = 1, E_NEGIDX = 2, E_TOGGLE_OVF = 4 };
enum Src { SRC_LABELS = 0, SRC_DENSE = 1 };
enum Out { OUT_U = 0, OUT_CH8 = 1 };

// Per-cartogram run state, device resident (engine.py:182-219 loop variables).
struct Carto {
    int active;         // 1 while the run continues
    int next_iter;      // iteration index of the next state to evaluate
    int best_iter;      // engine.py:196-199
    int best_pending;   // state (next_iter-1) is the new best: copy its vertices on the next advect
    int stop;           // Stop
    int collapsed;      // first zero-count region (engine.py:148-150)
    int err;            // Err bits
    int final_pending;  // stagnation: re-evaluate best vertices (engine.py:203-208)
    int res_iter;       // iteration of the returned state
    int trace_len;
    double best_xi;
    double eps, xi;
    double bdv, C;
    unsigned long long clamps;
    unsigned long long t_prev;
};

static_assert(sizeof(Carto) % 16 == 0, "k_region reads the first four state words as one int4");

// Per-cartogram constants (CartogramEngine.__init__, engine.py:98-141; StoppingCriteria).
struct Params {
    double background_mass, mult, mean_density0, S;
    double thr;
    int window, max_iter;
    int mode, pad;
};

struct Topo {
    int n_rows, R;
    const int* region_row0;   // R+1: first vertex row of each region (regions' rows are contiguous)
    const int* ring_start;    // n_rings+1: first vertex row of each ring
    const int* region_ring0;  // R+1: first ring of each region (a region's rings are contiguous)
    const int* region_rank;   // R: rank of region in ascending region_id order
    const int* rank_region;   // R: inverse
    const int* row_next;      // n_rows: next row of the same ring (wraps) -- multi-ring regions
    const int* row_uniq;      // n_rows: unique-vertex index of each row (unique-vertex state, k_region<.., UQ>)
};

struct Bufs {
    int B, n, k, cap, H, nb;
    int b0;           // first cartogram of this launch (frame groups run as parallel graph branches)
    size_t nn;
    // vertex rows (state, advected in place, + best state): double2 on the float64-field path,
    // float2 on the float32-field path (k_region<UT> reads them as Vec2<UT>)
    void* pos0;
    void* best;
    // unique-vertex state of the float64 graph iterations (one double2 per unique vertex and cartogram;
    // gathered from / expanded to the rows at the ends of each graph launch), its best copy, and a
    // per-cartogram flag word: 2 = gathered by this launch, 1 = ubest written
    double2* upos;
    double2* ubest;
    int* uq_flag;
    int n_uniq;
    // band-fused advect: per unique vertex the band (of H rows) holding both rows of its bilinear tap,
    // 255 when the tap straddles two bands; double-buffered by iteration parity (read [par], write [par^1]);
    // uq_bstride = per-cartogram stride (n_uniq rounded up to 16, pad bytes 254)
    unsigned char* uq_band[2];
    int uq_bstride;
    int* labels;
    int* cnt_acc;
    int* cnt_state;
    unsigned long long* spans;
    int* rowcnt;
    int* maxspan;
    int* rowdone;     // B: k_row CTAs finished this iteration (last one runs the control step)
    double* lut;
    float* lutf;      // float copy of lut for the float32-field band kernels
    const double* stats;
    const double* weights;
    double* rerr;
    void* uf;
    // integral-image partials / carries
    double* cs;    // B*nb*n
    double* dgc;   // B*nb*(n+H-1)
    double* adc;   // B*nb*(n+H-1)
    double* rt;    // B*n
    double* csX;   // B*nb*n
    double* dgXc;  // B*nb*n
    double* adSc;  // B*nb*(n+H-1)
    double* csT;   // B*n
    double* dgT;   // B*(2n-1)
    double* adT;   // B*(2n-1)
    double* rowfull;  // B*(n+1)
    double* tab;      // B*nb*4*(n/W)*H: k_sat1w's per-row slice tables for k_sat3w (W = slice width)
    Carto* st;
    const Params* prm;
    double* trace;
    int trace_cap;
};

struct SatSrc {
    const double* d;  // dense density (SRC_DENSE) n*n per cartogram
    double scale, offset;
    double outscale;  // OUT_U: field = anchor combination * outscale (0 -> 1/(2m), residual form)
    double* ch8;      // OUT_CH8 destination: 8*n*n
};

__device__ __forceinline__ int clampi(long long v, int lo, int hi) {
    return (int)(v < lo ? lo : (v > hi ? hi : v));
}

// Exact ceil / floor of a double as int without the conversion (XU) pipe: adding
// 1.5*2^52 in round-up / round-down mode leaves ceil(v) / floor(v) in the low mantissa
// bits (valid for |v| < 2^31, the texture-coordinate range here).
constexpr double ROUND_MAGIC = 6755399441055744.0;
__device__ __forceinline__ int ceil_to_int(double v) {
    return (int)(unsigned)__double_as_longlong(__dadd_ru(v, ROUND_MAGIC));
}
__device__ __forceinline__ int floor_to_int(double v) {
    return (int)(unsigned)__double_as_longlong(__dadd_rd(v, ROUND_MAGIC));
}
// ceil(v) for a float with -1 < v < 2^22 (the scaled texture range): adding 1.5*2^23 in
// round-up mode leaves ceil(v) in the low mantissa bits -- FP32 pipe only
__device__ __forceinline__ int ceil_to_int_f(float v) {
    return __float_as_int(__fadd_ru(v, 12582912.0f)) - 0x4B400000;
}
__device__ __forceinline__ double floor_exact(double v) {  // floor(v) as a double, FP64 pipe only
    return __dsub_rn(__dadd_rd(v, ROUND_MAGIC), ROUND_MAGIC);
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ bool gate_open(const Carto* st, int gate) {
    if (gate == G_ACTIVE) return st->active != 0;
    if (gate == G_FINAL) return st->final_pending != 0;
    return true;
}

// ---- deterministic block reductions (blockDim.x multiple of 32) ----
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_down_sync(FULL, v, o));
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_down_sync(FULL, v, o));
    return v;
}

// op: 0 sum, 1 min, 2 max.  Result broadcast to every thread.
template <int OP, typename T>
__device__ T block_reduce(T v, T ident, T* sm /*>=33*/) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = OP == 0 ? warp_sum(v) : (OP == 1 ? warp_min(v) : warp_max(v));
    __syncthreads();
    if (lane == 0) sm[w] = v;
    __syncthreads();
    if (w == 0) {
        T x = lane < nw ? sm[lane] : ident;
        x = OP == 0 ? warp_sum(x) : (OP == 1 ? warp_min(x) : warp_max(x));
        if (lane == 0) sm[32] = x;
    }
    __syncthreads();
    return sm[32];
}

// Inclusive warp scan.
__device__ __forceinline__ double warp_incl_scan(double v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double t = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block exclusive scan of one value per thread; returns the exclusive prefix, total in *tot.
__device__ double block_excl_scan(double v, double* sm /*>=33*/, double* tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    double inc = warp_incl_scan(v);
    __syncthreads();
    if (lane == 31) sm[w] = inc;
    __syncthreads();
    if (w == 0) {
        double x = lane < nw ? sm[lane] : 0.0;
        double xi = warp_incl_scan(x);
        if (lane < nw) sm[lane] = xi - x;  // exclusive warp offsets
        if (lane == 31) sm[32] = xi;
    }
    __syncthreads();
    double r = sm[w] + inc - v;
    *tot = sm[32];
    __syncthreads();
    return r;
}

// Inclusive prefix of in[0..len) (global, read via L1); stores prefix[i] to out[i - lo] for
// i in [lo, hi).  Indices below 0 are not representable: callers pass lo >= 0.
__device__ void block_prefix_window(const double* __restrict__ in, int len, double* out, int lo, int hi,
                                    double* sm) {
    const int nt = blockDim.x;
    const int per = (len + nt - 1) / nt;
    const int a = min(len, threadIdx.x * per), e = min(len, a + per);
    double s = 0.0;
    for (int i = a; i < e; ++i) s += __ldg(in + i);
    double tot;
    double run = block_excl_scan(s, sm, &tot);
    for (int i = a; i < e; ++i) {
        run += __ldg(in + i);
        if (i >= lo && i < hi) out[i - lo] = run;
    }
}

}  // namespace det
