// Advection + rasterisation kernels (sm_100a).
//
// Vertex positions live per ring row (the order of MapModel.vertex_array(),
// geomodel.py:128-130), so every region's rows are one contiguous, coalesced
// range.  Rows that duplicate a shared vertex evolve bit-identically (same input,
// same arithmetic), exactly as in the reference.
//
// k_region : one WARP per (region, cartogram), no CTA-wide barriers.  Fuses
//            * advect (displacement.py:209-238): bilinear sample of the u field at
//              every vertex row, clamp to [0,1]^2, clamp count;
//            * the region's bounding-box crop (raster.py:70-78);
//            * even-odd crossing toggles of every ring edge (raster.py:23-61) with the
//              reference's exact float64 op order (explicit _rn intrinsics, no FMA);
//            * the crop flattening of _submask incl. the absorber column and the
//              negative-index case (raster.py:79-90);
//            * a counting sort of the toggles by row and even-odd pairing into spans
//              (start, end, rank) appended to per-row buckets in HBM;
//            * the region's provisional pixel count = sum of its span lengths.
// k_row    : one WARP per (texture row, cartogram).  Paints spans with smem atomicMin
//            on the region rank (ascending-id first-writer-wins, raster.py:142-146);
//            every lost claim decrements the loser's count, so counts are exact
//            (raster.py:110-118); writes the label row (BACKGROUND=-1).  The last CTA
//            of a cartogram derives the background count and runs the control step
//            (det_ctrl.cuh) -- no separate launch.
#pragma once
#include <type_traits>
#include "det_common.cuh"
#include "det_ctrl.cuh"

namespace det {

#ifndef DET_RW_WARPS
#define DET_RW_WARPS 2  // 1, 2, 4 measured: 2 frees slots of finished regions sooner without over-splitting
#endif
constexpr int RW_WARPS = DET_RW_WARPS;  // warps (regions) per CTA
#ifndef DET_RW_ROWCAP
#define DET_RW_ROWCAP 384
#endif
constexpr int RW_ROWCAP = DET_RW_ROWCAP;  // vertex rows kept in smem per warp (288 with 16-bit jr: 1% slower)
constexpr int RW_TCAP = 256;     // toggles per warp window
constexpr int RW_WROWS = 128;    // texture rows per warp window
#ifndef DET_RW_PIPE
#define DET_RW_PIPE 1
#endif
#ifndef DET_RW_UNROLL
#define DET_RW_UNROLL 2
#endif
#ifndef DET_RW_UNROLL_RO
#define DET_RW_UNROLL_RO 5  // raster-only k_region (2: 55.5k, 3: 56.0k, 4: 56.25k, 5: 56.4k, 6: 56.4k, 8: 55.2k it/s)
#endif
constexpr int RW_UNROLL_RO = DET_RW_UNROLL_RO;
constexpr int RW_UNROLL = DET_RW_UNROLL;  // vertex rows in flight per lane (2 measured best of 1-8)

// Bilinear sample of the field (displacement.py:209-226): g = p*n - 0.5,
// i0 = clip(floor(g), 0, n-2), f = clip(g - i0, 0, 1), 4-tap blend.  Index math in
// float64; a float32 field is blended in float32 (its own precision), so the eight
// texels need no float->double conversions.
struct Tap {
    int o0, o1;      // element offsets of the two texel pairs
    double fx, fy;
};

__device__ __forceinline__ Tap field_tap(int n, double px, double py) {
    const double nd = (double)n;
    const double gx = px * nd - 0.5, gy = py * nd - 0.5;
    const double hi = (double)(n - 2);
    double bx = floor_exact(gx), by = floor_exact(gy);
    bx = bx < 0.0 ? 0.0 : (bx > hi ? hi : bx);
    by = by < 0.0 ? 0.0 : (by > hi ? hi : by);
    const int ix = floor_to_int(bx), iy = floor_to_int(by);
    Tap t;
    t.fx = gx - bx;
    t.fy = gy - by;
    t.fx = t.fx < 0.0 ? 0.0 : (t.fx > 1.0 ? 1.0 : t.fx);
    t.fy = t.fy < 0.0 ? 0.0 : (t.fy > 1.0 ? 1.0 : t.fy);
    t.o0 = (iy * n + ix) * 2;
    t.o1 = t.o0 + n * 2;
    return t;
}

// Float-field tap: the fraction only feeds a float blend, so floor / clamp / fraction run in
// float32 after one float64 FMA.  The texel choice can differ from the float64 rule only where
// the fraction is within float rounding of 0 or 1, where both neighbours blend to the same value.
struct TapF {
    int o0, o1;
    float fx, fy;
};

__device__ __forceinline__ TapF field_tap_f(int n, double px, double py) {
    constexpr float M = 12582912.0f;  // 1.5 * 2^23: x + M rounded down holds floor(x) in its low bits
    const float gx = (float)fma(px, (double)n, -0.5), gy = (float)fma(py, (double)n, -0.5);
    const float tx = __fadd_rd(gx, M), ty = __fadd_rd(gy, M);
    const int ix = min(max(__float_as_int(tx) - 0x4B400000, 0), n - 2);
    const int iy = min(max(__float_as_int(ty) - 0x4B400000, 0), n - 2);
    const float hi = (float)(n - 2);
    TapF t;
    t.fx = __saturatef(gx - fminf(fmaxf(tx - M, 0.0f), hi));
    t.fy = __saturatef(gy - fminf(fmaxf(ty - M, 0.0f), hi));
    t.o0 = (iy * n + ix) * 2;
    t.o1 = t.o0 + n * 2;
    return t;
}

template <typename UT>
struct Texels {
    UT v[8];
};

template <typename UT>
struct Vec2;
template <>
struct Vec2<float> {
    using type = float2;
};
template <>
struct Vec2<double> {
    using type = double2;
};

// the four texels as (u, v) pairs: one 8-byte (float) / 16-byte (double) load each
template <typename UT, typename TP>
__device__ __forceinline__ Texels<UT> field_load(const UT* __restrict__ uf, const TP& t) {
    using V = typename Vec2<UT>::type;
    const V* __restrict__ u2 = reinterpret_cast<const V*>(uf);
    const V a = __ldg(u2 + (t.o0 >> 1)), b = __ldg(u2 + (t.o0 >> 1) + 1);
    const V c = __ldg(u2 + (t.o1 >> 1)), d = __ldg(u2 + (t.o1 >> 1) + 1);
    Texels<UT> x;
    x.v[0] = a.x; x.v[1] = a.y; x.v[2] = b.x; x.v[3] = b.y;
    x.v[4] = c.x; x.v[5] = c.y; x.v[6] = d.x; x.v[7] = d.y;
    return x;
}

// the four texels with plain (coherent) loads: for a field written earlier by this same kernel
// (band-fused advect), where the read-only path of field_load must not be used
__device__ __forceinline__ Texels<double> field_load_coherent(const double* uf, const Tap& t) {
    const double2* u2 = reinterpret_cast<const double2*>(uf);
    const double2 a = u2[t.o0 >> 1], b = u2[(t.o0 >> 1) + 1];
    const double2 c = u2[t.o1 >> 1], d = u2[(t.o1 >> 1) + 1];
    Texels<double> x;
    x.v[0] = a.x; x.v[1] = a.y; x.v[2] = b.x; x.v[3] = b.y;
    x.v[4] = c.x; x.v[5] = c.y; x.v[6] = d.x; x.v[7] = d.y;
    return x;
}

// Band of H rows (H = 1 << lgH) holding BOTH rows iy, iy + 1 of the bilinear tap of a vertex at
// height py (field_tap's row: iy = clip(floor(py*n - 0.5), 0, n-2)); 255 when iy is a band's last
// row, so that the tap straddles two bands.
__device__ __forceinline__ unsigned char tap_band(int n, int lgH, double py) {
    const double gy = py * (double)n - 0.5;
    const double hi = (double)(n - 2);
    double by = floor_exact(gy);
    by = by < 0.0 ? 0.0 : (by > hi ? hi : by);
    const int iy = floor_to_int(by);
    const int H = 1 << lgH;
    return (unsigned char)(((iy & (H - 1)) == H - 1) ? 255 : (iy >> lgH));
}

template <typename UT, typename TP>
__device__ __forceinline__ double2 field_blend(const Texels<UT>& x, const TP& t) {
    const UT fx = (UT)t.fx, fy = (UT)t.fy;
    const UT gxm = (UT)1 - fx, gym = (UT)1 - fy;
    const UT sx = x.v[0] * gxm * gym + x.v[2] * fx * gym + x.v[4] * gxm * fy + x.v[6] * fx * fy;
    const UT sy = x.v[1] * gxm * gym + x.v[3] * fx * gym + x.v[5] * gxm * fy + x.v[7] * fx * fy;
    return make_double2((double)sx, (double)sy);
}

// float state path: the same blend, result kept in float (the position update is a float add)
__device__ __forceinline__ float2 field_blend_f(const Texels<float>& x, const TapF& t) {
    const float gxm = 1.0f - t.fx, gym = 1.0f - t.fy;
    const float sx = x.v[0] * gxm * gym + x.v[2] * t.fx * gym + x.v[4] * gxm * t.fy + x.v[6] * t.fx * t.fy;
    const float sy = x.v[1] * gxm * gym + x.v[3] * t.fx * gym + x.v[5] * gxm * t.fy + x.v[7] * t.fx * t.fy;
    return make_float2(sx, sy);
}

// Tap of a float position: p*n is exact (n a power of two) and p*n - 0.5 is exact whenever it is
// >= -0.25, so one FMA gives the reference's g; below that the tap clamps to column/row 0 with
// fraction 0 either way.
__device__ __forceinline__ TapF field_tap_pf(int n, float px, float py) {
    constexpr float M = 12582912.0f;
    const float nf = (float)n;
    const float gx = fmaf(px, nf, -0.5f), gy = fmaf(py, nf, -0.5f);
    const float tx = __fadd_rd(gx, M), ty = __fadd_rd(gy, M);
    const int ix = min(max(__float_as_int(tx) - 0x4B400000, 0), n - 2);
    const int iy = min(max(__float_as_int(ty) - 0x4B400000, 0), n - 2);
    const float hi = (float)(n - 2);
    TapF t;
    t.fx = __saturatef(gx - fminf(fmaxf(tx - M, 0.0f), hi));
    t.fy = __saturatef(gy - fminf(fmaxf(ty - M, 0.0f), hi));
    t.o0 = (iy * n + ix) * 2;
    t.o1 = t.o0 + n * 2;
    return t;
}

__device__ __forceinline__ double2 to_d2(const double2& p) { return p; }
__device__ __forceinline__ double2 to_d2(const float2& p) { return make_double2((double)p.x, (double)p.y); }

template <typename UT>
__device__ __forceinline__ double2 sample_field(const UT* __restrict__ uf, int n, double px, double py) {
    const Tap t = field_tap(n, px, py);
    return field_blend<UT>(field_load<UT>(uf, t), t);
}

template <typename T>
__device__ __forceinline__ T warp_allmin(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_allmax(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

__device__ __forceinline__ int warp_excl_scan_int(int v, int lane, int* total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    *total = __shfl_sync(FULL, x, 31);
    return x - v;
}

// UT: field element type (float / double); ST: vertex-state element type.  <float, float> is the
// float32 path, <double, double> the float64 path, <float, double> the mixed path (float32 field,
// float64 state and position update).
template <typename UT, typename ST = UT, bool BM = false, bool ADV = true, bool UQ = false>
#ifndef DET_RW_MINB
#define DET_RW_MINB (32 / DET_RW_WARPS)  // 32 resident warps per SM (64 registers)
#endif
#ifndef DET_RW_MINB64
#define DET_RW_MINB64 (24 / DET_RW_WARPS)  // float64 state: 24 warps per SM (80 registers)
#endif
#ifndef DET_RW_MINB_RO
#define DET_RW_MINB_RO (32 / DET_RW_WARPS)  // raster-only instantiation: 64 registers, 32 warps per SM
#endif
// ADV = false: the raster-only instantiation (the advect phase compiled out, fewer registers, more
// warps per SM) for launches without M_ADVECT: start / final rasters and the split advect path.
__global__ void __launch_bounds__(RW_WARPS * 32, ADV ? (sizeof(ST) == 8 ? DET_RW_MINB64 : DET_RW_MINB) : DET_RW_MINB_RO)
    k_region(Topo T, Bufs D, int mode_in, int gate, int src) {
    const int mode = ADV ? mode_in : (mode_in & ~(int)M_ADVECT);
    // per row: ceil(y*n - 0.5) clipped to [0, n] (low 16 bits) | next row of the same ring,
    // region-local (high 16 bits) -- one load per edge end
    __shared__ uint32_t s_jn[RW_WARPS][RW_ROWCAP];
    __shared__ int s_tot[RW_WARPS];
    __shared__ uint32_t s_key[RW_WARPS][RW_TCAP];
    __shared__ uint16_t s_col[RW_WARPS][RW_TCAP];
    __shared__ __align__(16) int s_rc[RW_WARPS][RW_WROWS + 4];  // 16-byte rows: zeroed as int4
    __shared__ uint32_t s_q[RW_WARPS][64];  // compacted crossing edges (ring buffer)

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r = blockIdx.x * RW_WARPS + wid, b = blockIdx.y + D.b0;
    if (r >= T.R) return;
    Carto* st = D.st + b;
    // the region's bounds and the cartogram's state words in one memory round trip, then the gate
    const int row0 = T.region_row0[r], row1 = T.region_row0[r + 1];
    const int rq0 = T.region_ring0[r], rq1 = T.region_ring0[r + 1];
    const int4 sth = *reinterpret_cast<const int4*>(st);  // active, next_iter, best_iter, best_pending
    if (gate == G_ACTIVE ? sth.x == 0 : (gate == G_FINAL && st->final_pending == 0)) return;
    const int n = D.n;
    const double nd = (double)n;
    const int nrows = row1 - row0;
    const size_t ub = (size_t)b * T.n_rows;
    const bool in_smem = nrows <= RW_ROWCAP;
    uint32_t* sjn = s_jn[wid];
    uint32_t* keys = s_key[wid];
    uint16_t* colb = s_col[wid];
    int* rc = s_rc[wid];

    // next row of the same ring (wraps): from the region's ring boundaries, no per-row table
    auto next_row = [&](int v) -> int {
        if (rq1 - rq0 == 1) return v + 1 < row1 ? v + 1 : row0;
        // a multi-ring region too large for shared memory (its edge scan repeats per toggle
        // window): the static successor table, O(1) per edge; smaller ones walk their rings once
        if (!in_smem) return __ldg(T.row_next + v);
        int q = rq0;
        while (T.ring_start[q + 1] <= v) ++q;
        const int e = T.ring_start[q + 1];
        return v + 1 < e ? v + 1 : T.ring_start[q];
    };

    // vertex rows: float64 on the float64 and mixed paths, float32 on the float32 path
    using PT = typename Vec2<ST>::type;
    constexpr bool FS = sizeof(ST) == 4;
    // the state rows live in pos0 and are advected IN PLACE: each row is read and rewritten by the
    // same lane, and other lanes read it only after a __syncwarp (no ping-pong, so the buffer
    // does not depend on the iteration counter and the row loads need no state round trip)
    PT* __restrict__ pbest = reinterpret_cast<PT*>(D.best) + ub;
    const bool bestcopy = (mode & M_ADVECT) && sth.w != 0;
    PT* const pin = reinterpret_cast<PT*>((mode & (M_ADVECT | M_POSTADV)) || src == 0 ? D.pos0 : D.best) + ub;
    PT* const pout = pin;
    // UQ (raster-only, float64): the rows' positions come from the unique-vertex state through the
    // static row -> unique-vertex table (the rows themselves are stale inside a graph launch)
    const double2* upos = UQ ? D.upos + (size_t)b * D.n_uniq : nullptr;
    auto rowpos = [&](int v) -> PT {
        if constexpr (UQ) {
            const double2 q = upos[__ldg(T.row_uniq + v)];
            return PT{(ST)q.x, (ST)q.y};
        } else {
            return pin[v];
        }
    };
    const UT* uf = reinterpret_cast<const UT*>(D.uf) + (size_t)b * D.nn * 2;

    // ---- phase A: advect every vertex row (Q rows in flight per lane); per-row scaled
    //      coordinates and scanline / column indices for the raster ----
    int jmn = n, jmx = 0, imn = n, imx = 0;
    int ncl = 0;
    // per advected row: store (in place), best copy, scanline / column index, crop extent
    auto finish = [&](int v, const PT& pold, const PT& pnew) {
        if (mode & M_ADVECT) {
            pout[v] = pnew;
            if (bestcopy) pbest[v] = pold;
        }
        // x*n, y*n are exact (n is a power of two); ceil is monotone, so the crop
        // (raster.py:71-74) and each edge's scanline range (raster.py:45-46) are
        // min/max of these per-row integers
        int jr, ir;
        if constexpr (FS) {  // y*n - 0.5 is exact in float wherever its ceil is not 0
            const float nf = (float)n;
            jr = min(max(ceil_to_int_f(pnew.y * nf - 0.5f), 0), n);
            ir = min(max(ceil_to_int_f(pnew.x * nf - 0.5f), 0), n);
        } else {
            const double xs = __dmul_rn(pnew.x, nd), ys = __dmul_rn(pnew.y, nd);
            jr = min(max(ceil_to_int(__dsub_rn(ys, 0.5)), 0), n);
            ir = min(max(ceil_to_int(__dsub_rn(xs, 0.5)), 0), n);
        }
        if (in_smem) {
            sjn[v - row0] = (uint32_t)jr | ((uint32_t)(next_row(v) - row0) << 16);
        }
        jmn = min(jmn, jr); jmx = max(jmx, jr);
        imn = min(imn, ir); imx = max(imx, ir);
    };
    auto chunk = [&](auto QC, int base) {
        constexpr int Q = decltype(QC)::value;
        PT p[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int v = base + q * 32 + lane;
            p[q] = v < row1 ? rowpos(v) : PT{0.5, 0.5};
        }
        PT nq[Q];
        if (mode & M_ADVECT) {
            if constexpr (FS) {
                // float state: tap, blend, update and clamp in float32
                TapF tp[Q];
                Texels<float> tx[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    tp[q] = field_tap_pf(n, p[q].x, p[q].y);
                    tx[q] = field_load<float, TapF>(reinterpret_cast<const float*>(uf), tp[q]);
                }
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const float2 s = field_blend_f(tx[q], tp[q]);
                    const float mx = p[q].x + s.x, my = p[q].y + s.y;
                    const float cx = mx < 0.0f ? 0.0f : (mx > 1.0f ? 1.0f : mx);  // np.clip (no NaNs here)
                    const float cy = my < 0.0f ? 0.0f : (my > 1.0f ? 1.0f : my);
                    const int v = base + q * 32 + lane;
                    if (v < row1) ncl += (cx != mx) + (cy != my);
                    nq[q] = PT{cx, cy};
                }
            } else {
                Tap tp[Q];
                Texels<UT> tx[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    tp[q] = field_tap(n, (double)p[q].x, (double)p[q].y);
                    tx[q] = field_load<UT, Tap>(uf, tp[q]);
                }
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const double2 s = field_blend<UT, Tap>(tx[q], tp[q]);
                    const double mx = p[q].x + s.x, my = p[q].y + s.y;
                    const double cx = mx < 0.0 ? 0.0 : (mx > 1.0 ? 1.0 : mx);  // np.clip (no NaNs here)
                    const double cy = my < 0.0 ? 0.0 : (my > 1.0 ? 1.0 : my);
                    const int v = base + q * 32 + lane;
                    if (v < row1) ncl += (cx != mx) + (cy != my);
                    nq[q] = PT{cx, cy};
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < Q; ++q) nq[q] = p[q];
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int v = base + q * 32 + lane;
            if (v < row1) finish(v, p[q], nq[q]);
        }
    };
    // full rounds of RW_UNROLL rows per lane while more than one warp of rows remains, then a
    // one-row tail (no lane slots idle for a whole extra round)
    bool done_a = false;
#if DET_RW_PIPE
    if (mode & M_ADVECT) {
        // software-pipelined advect: the next chunk's row loads are issued together with this
        // chunk's texel gather, so a region pays one round trip per chunk, not two
        constexpr int Q = RW_UNROLL;
        PT pc[Q], pn[Q];
        auto ld = [&](PT (&dst)[Q], int base) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int v = base + q * 32 + lane;
                dst[q] = v < row1 ? pin[v] : PT{0.5, 0.5};
            }
        };
        ld(pc, row0);
        for (int base = row0; base < row1; base += 32 * Q) {
            if constexpr (FS) {  // float state: tap, blend, update and clamp in float32
                TapF tp[Q];
                Texels<float> tx[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    tp[q] = field_tap_pf(n, pc[q].x, pc[q].y);
                    tx[q] = field_load<float, TapF>(reinterpret_cast<const float*>(uf), tp[q]);
                }
                if (base + 32 * Q < row1) ld(pn, base + 32 * Q);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const float2 sm = field_blend_f(tx[q], tp[q]);
                    const float mx = pc[q].x + sm.x, my = pc[q].y + sm.y;
                    const float cx = mx < 0.0f ? 0.0f : (mx > 1.0f ? 1.0f : mx);  // np.clip (no NaNs here)
                    const float cy = my < 0.0f ? 0.0f : (my > 1.0f ? 1.0f : my);
                    const int v = base + q * 32 + lane;
                    if (v < row1) {
                        ncl += (cx != mx) + (cy != my);
                        finish(v, pc[q], make_float2(cx, cy));
                    }
                }
            } else {  // float64 state: float64 tap and update (displacement.py:209-238 op order)
                Tap tp[Q];
                Texels<UT> tx[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    tp[q] = field_tap(n, (double)pc[q].x, (double)pc[q].y);
                    tx[q] = field_load<UT, Tap>(uf, tp[q]);
                }
                if (base + 32 * Q < row1) ld(pn, base + 32 * Q);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const double2 sm = field_blend<UT, Tap>(tx[q], tp[q]);
                    const double mx = pc[q].x + sm.x, my = pc[q].y + sm.y;
                    const double cx = mx < 0.0 ? 0.0 : (mx > 1.0 ? 1.0 : mx);  // np.clip (no NaNs here)
                    const double cy = my < 0.0 ? 0.0 : (my > 1.0 ? 1.0 : my);
                    const int v = base + q * 32 + lane;
                    if (v < row1) {
                        ncl += (cx != mx) + (cy != my);
                        finish(v, pc[q], PT{cx, cy});
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) pc[q] = pn[q];
        }
        done_a = true;
    }
#endif
    if (!done_a) {
        // raster-only instantiations keep RW_UNROLL_RO rows in flight per lane (no advect state to hold)
        constexpr int RU = ADV ? RW_UNROLL : RW_UNROLL_RO;
        int base = row0;
        for (; base + 32 < row1; base += 32 * RU) chunk(std::integral_constant<int, RU>{}, base);
        if (base < row1) chunk(std::integral_constant<int, 1>{}, base);
    }
    if (mode & M_ADVECT) {
        ncl = warp_sum(ncl);
        if (lane == 0 && ncl) atomicAdd(&st->clamps, (unsigned long long)ncl);
    }
    if (!(mode & M_RASTER)) return;
    const int j_off = warp_allmin(jmn), j_end = warp_allmax(jmx);
    const int i_off = warp_allmin(imn), i_end = warp_allmax(imx);
    __syncwarp();  // row data (smem, or this warp's global writes) visible to the warp

    int* cnt = D.cnt_acc + (size_t)b * (T.R + 1);
    const int rows = max(j_end - j_off, 0), cols = max(i_end - i_off, 0);
    if (rows == 0 || cols == 0) {
        if (lane == 0) cnt[r] = 0;
        return;
    }
    const long long width = (long long)cols + 1;  // absorber column (raster.py:79-80)
    const unsigned long long rank = (unsigned long long)T.region_rank[r];
    // max rows a negative column moves a toggle up: i_off / (cols + 1) + 1, the quotient from a
    // float reciprocal (exact to +-1 for these magnitudes) corrected with one integer product
    int back;
    {
        const int w1 = cols + 1;
        int q = (int)((float)i_off * __frcp_rn((float)w1));
        q -= q * w1 > i_off;
        q += (q + 1) * w1 <= i_off;
        back = q + 1;
    }
    int area = 0;

    // BM: one scanline j of this region rasterised through a parity bitmap of its crop columns
    // (keys[] reused: RW_TCAP words = 8192 bits >= cols), for any number of crossings -- the
    // bincount of raster.py:80-89 has no limit.  Every edge is re-scanned from the global rows
    // with emit()'s exact arithmetic; a column's bit is the parity of its toggles, pixel c is
    // inside iff the inclusive prefix XOR at c is 1 (cumsum & 1, raster.py:86-89), and runs of
    // inside pixels become spans (split at 32-column words; painting and counts are per pixel).
    auto bitmap_row = [&](int jrow) -> int {
        for (int q = lane; q < RW_TCAP; q += 32) keys[q] = 0u;
        __syncwarp();
        for (int e = row0 + lane; e < row1; e += 32) {
            const int en = __ldg(T.row_next + e);
            double2 a = to_d2(rowpos(e)), c = to_d2(rowpos(en));
            const int ja = min(max(ceil_to_int(__dsub_rn(__dmul_rn(a.y, nd), 0.5)), 0), n);
            const int jb2 = min(max(ceil_to_int(__dsub_rn(__dmul_rn(c.y, nd), 0.5)), 0), n);
            const int js = max(min(ja, jb2), jrow), je = min(max(ja, jb2), jrow + 1 + back);
            if (je <= js) continue;
            a = make_double2(__dmul_rn(a.x, nd), __dmul_rn(a.y, nd));
            c = make_double2(__dmul_rn(c.x, nd), __dmul_rn(c.y, nd));
            const double slope = __ddiv_rn(__dsub_rn(c.x, a.x), __dsub_rn(c.y, a.y));
            double yc = (double)js + 0.5;
            for (int j = js; j < je; ++j, yc += 1.0) {
                const double xc = __dadd_rn(a.x, __dmul_rn(__dsub_rn(yc, a.y), slope));
                const int i0 = min(max(ceil_to_int(__dsub_rn(xc, 0.5)), 0), n);
                int dest = j, cc = min(i0 - i_off, cols);
                if (cc < 0) {
                    const long long f = (long long)(j - j_off) * width + (long long)cc;
                    if (f < 0) continue;  // flagged (E_NEGIDX) by the windowed pass already
                    const long long dr = f / width;
                    cc = (int)(f - dr * width);
                    dest = j_off + (int)dr;
                }
                if (cc == cols || dest != jrow) continue;
                atomicXor(&keys[cc >> 5], 1u << (cc & 31));
            }
        }
        __syncwarp();
        const int nw = (cols + 31) >> 5;
        const size_t rb = (size_t)b * n + jrow;
        int px = 0, carry = 0, slot = 0;
        for (int pass = 0; pass < 2; ++pass) {  // pass 0 counts spans, pass 1 writes them
            int nsp_all = 0;
            carry = 0;
            for (int q0 = 0; q0 < nw; q0 += 32) {
                const int q = q0 + lane;
                const uint32_t x = q < nw ? keys[q] : 0u;
                uint32_t pfx = x;
                pfx ^= pfx << 1; pfx ^= pfx << 2; pfx ^= pfx << 4; pfx ^= pfx << 8; pfx ^= pfx << 16;
                const unsigned par = __ballot_sync(FULL, __popc(x) & 1);
                const int pre = (carry + __popc(par & ((1u << lane) - 1u))) & 1;
                carry = (carry + __popc(par)) & 1;
                uint32_t in = pre ? ~pfx : pfx;
                if (q >= nw) in = 0u;
                else if (cols - q * 32 < 32) in &= (1u << (cols - q * 32)) - 1u;
                const int nsp = __popc(in & ~(in << 1));
                if (pass == 0) {
                    nsp_all += nsp;
                    continue;
                }
                int chunk;
                int sl = slot + warp_excl_scan_int(nsp, lane, &chunk);
                slot += chunk;
                px += __popc(in);
                while (in) {
                    const int lo = __ffs(in) - 1;
                    const uint32_t rest = ~(in | ((1u << lo) - 1u));
                    const int hi = rest ? __ffs(rest) - 1 : 32;
                    in = hi < 32 ? (in & ~((1u << hi) - 1u)) : 0u;
                    if (sl < D.cap)
                        D.spans[rb * D.cap + sl] = (rank << 32) | ((unsigned long long)(i_off + q * 32 + hi) << 16) |
                                                   (unsigned long long)(i_off + q * 32 + lo);
                    else
                        atomicOr(&st->err, (int)E_SPAN_OVF);
                    ++sl;
                }
            }
            if (pass == 0) {
                nsp_all = warp_sum(nsp_all);
                int base = 0;
                if (lane == 0 && nsp_all) base = atomicAdd(&D.rowcnt[rb], nsp_all);
                slot = __shfl_sync(FULL, base, 0);
            }
        }
        __syncwarp();
        return px;
    };
    int w0 = j_off, wh = min(rows, RW_WROWS);
    while (w0 < j_end) {
        const int w1 = min(w0 + wh, j_end);
        const int W = w1 - w0;
        for (int q = lane; q <= (W >> 2); q += 32) reinterpret_cast<int4*>(rc)[q] = make_int4(0, 0, 0, 0);
        __syncwarp();
        // ---- crossings of every ring edge (raster.py:30-61, flattening :86-89) ----
        if (lane == 0) s_tot[wid] = 0;
        __syncwarp();
        // toggles of one edge a -> c crossing scanlines [js, je) (raster.py:45-61)
        auto emit = [&](double2 a, double2 c, int js, int je) {
            a = make_double2(__dmul_rn(a.x, nd), __dmul_rn(a.y, nd));
            c = make_double2(__dmul_rn(c.x, nd), __dmul_rn(c.y, nd));
            const double x0 = a.x, y0 = a.y;
            const double slope = __ddiv_rn(__dsub_rn(c.x, a.x), __dsub_rn(c.y, a.y));
            double yc = (double)js + 0.5;  // scanline centre j + 0.5 (exact, stepped by 1.0)
            for (int j = js; j < je; ++j, yc += 1.0) {
                const double xc = __dadd_rn(x0, __dmul_rn(__dsub_rn(yc, y0), slope));
                const int i0 = min(max(ceil_to_int(__dsub_rn(xc, 0.5)), 0), n);
                int dest = j, cc = min(i0 - i_off, cols);
                if (cc < 0) {  // toggle left of the crop: the flat index lands in an earlier row
                    const long long f = (long long)(j - j_off) * width + (long long)cc;
                    if (f < 0) {  // np.bincount raises on negative entries
                        atomicOr(&st->err, (int)E_NEGIDX);
                        continue;
                    }
                    const long long dr = f / width;
                    cc = (int)(f - dr * width);
                    dest = j_off + (int)dr;
                }
                if (cc == cols || dest < w0 || dest >= w1) continue;  // absorber column / other window
                const int slot = atomicAdd(&s_tot[wid], 1);
                if (slot < RW_TCAP) {
                    keys[slot] = ((uint32_t)(dest - w0) << 16) | (uint32_t)(i_off + cc);
                    atomicAdd(&rc[dest - w0], 1);
                }
            }
        };
        if (in_smem) {
            // edges that cross a scanline centre (~30%) are compacted into a ring queue and
            // processed 32 at a time, so the float64 crossing work runs on full warps
            uint32_t* q = s_q[wid];
            int qh = 0, qt = 0;
            auto run = [&](uint32_t ent) {
                const int el = (int)(ent & 0xFFFFu), en = (int)(ent >> 16);
                const int ja = (int)(sjn[el] & 0xFFFFu), jb2 = (int)(sjn[en] & 0xFFFFu);
                emit(to_d2(rowpos(row0 + el)), to_d2(rowpos(row0 + en)), max(min(ja, jb2), w0), min(max(ja, jb2), w1 + back));
            };
            for (int e0 = 0; e0 < nrows; e0 += 32) {
                const int el = e0 + lane;
                bool cr = false;
                int en = 0;
                if (el < nrows) {
                    const uint32_t jl = sjn[el];
                    en = (int)(jl >> 16);
                    const int ja = (int)(jl & 0xFFFFu), jb2 = (int)(sjn[en] & 0xFFFFu);
                    cr = min(max(ja, jb2), w1 + back) > max(min(ja, jb2), w0);
                }
                const unsigned m = __ballot_sync(FULL, cr);
                if (cr) q[(qt + __popc(m & ((1u << lane) - 1u))) & 63] = (uint32_t)el | ((uint32_t)en << 16);
                qt += __popc(m);
                __syncwarp();
                if (qt - qh >= 32) {
                    run(q[(qh + lane) & 63]);
                    qh += 32;
                    __syncwarp();
                }
            }
            if (lane < qt - qh) run(q[(qh + lane) & 63]);
        } else {
            for (int e = row0 + lane; e < row1; e += 32) {
                const int en = next_row(e) - row0;
                const double2 a = to_d2(rowpos(e)), c = to_d2(rowpos(row0 + en));
                const int ja = min(max(ceil_to_int(__dsub_rn(__dmul_rn(a.y, nd), 0.5)), 0), n);
                const int jb2 = min(max(ceil_to_int(__dsub_rn(__dmul_rn(c.y, nd), 0.5)), 0), n);
                const int js = max(min(ja, jb2), w0);  // scanlines j in [jlo, jhi) are crossed
                const int je = min(max(ja, jb2), w1 + back);
                if (je > js) emit(a, c, js, je);
            }
        }
        __syncwarp();
        const int tot = s_tot[wid];
        __syncwarp();
        if (tot > RW_TCAP) {
            if (W == 1) {
                if constexpr (BM) {
                    // more toggles on scanline w0 than the key buffer holds: the parity-bitmap
                    // slow path (only in the BM instantiation the host switches to on overflow)
                    area += bitmap_row(w0);
                    w0 = w1;
                    __syncwarp();
                    continue;
                } else {
                    if (lane == 0) atomicOr(&st->err, (int)E_TOGGLE_OVF);
                    return;
                }
            }
            wh = max(1, W >> 1);
            __syncwarp();
            continue;
        }
        // ---- counting sort by row: rc -> exclusive offsets ----
        {
            int carry = 0;
            for (int q0 = 0; q0 < W; q0 += 32) {
                const int q = q0 + lane;
                const int v = q < W ? rc[q] : 0;
                int chunk;
                const int ex = warp_excl_scan_int(v, lane, &chunk);
                __syncwarp();
                if (q < W) rc[q] = carry + ex;
                carry += chunk;
            }
        }
        __syncwarp();
        // reserve every row's span slots now -- each row of crossings pairs into (c+1)/2 spans --
        // so the global atomics' latency overlaps the scatter and the sort below
        constexpr int RW_QPL = RW_WROWS / 32;  // rows per lane
        int sbase[RW_QPL];
#pragma unroll
        for (int u = 0; u < RW_QPL; ++u) {
            const int q = lane + 32 * u;
            sbase[u] = 0;
            if (q < W) {
                const int c = (q + 1 < W ? rc[q + 1] : tot) - rc[q];
                if (c > 0) sbase[u] = atomicAdd(&D.rowcnt[(size_t)b * n + w0 + q], (c + 1) >> 1);
            }
        }
        // scatter columns into row buckets; a bucket's cursor runs from its start to the next start
        for (int p = lane; p < tot; p += 32) {
            const uint32_t key = keys[p];
            const int pos = atomicAdd(&rc[key >> 16], 1);
            colb[pos] = (uint16_t)(key & 0xFFFFu);
        }
        __syncwarp();
        // after the scatter rc[q] = end of bucket q = start of bucket q+1
#pragma unroll
        for (int u = 0; u < RW_QPL; ++u) {
            const int q = lane + 32 * u;
            if (q >= W) break;
            const int s = q == 0 ? 0 : rc[q - 1], e = rc[q];
            // insertion sort of the (few) crossings of this row, then even-odd pairing
            for (int i = s + 1; i < e; ++i) {
                const uint16_t x = colb[i];
                int k = i - 1;
                while (k >= s && colb[k] > x) { colb[k + 1] = colb[k]; --k; }
                colb[k + 1] = x;
            }
            const size_t rb = (size_t)b * n + w0 + q;
            int slot = sbase[u];
            for (int i = s; i < e; i += 2, ++slot) {
                const int col = colb[i];
                int end = i + 1 < e ? (int)colb[i + 1] : i_end;
                if (end > col) area += end - col;
                else end = col;  // empty pair: a zero-length span keeps the reserved slot valid
                if (slot < D.cap)
                    D.spans[rb * D.cap + slot] = (rank << 32) | ((unsigned long long)end << 16) | (unsigned long long)col;
                else
                    atomicOr(&st->err, (int)E_SPAN_OVF);
            }
        }
        __syncwarp();
        w0 = w1;
        if (tot < RW_TCAP / 4 && wh < RW_WROWS) wh = min(wh << 1, RW_WROWS);
    }
    area = warp_sum(area);
    if (lane == 0) cnt[r] = area;  // provisional; k_row subtracts pixels lost to lower ranks
}

// Advect as its own flat kernel (float32 state): ADV_RPT rows per thread over the whole row range
// of each cartogram (grid.y), every lane busy and ~64 warps per SM to cover the position -> texel
// load chain; the same float arithmetic as k_region's phase A (displacement.py:209-238).
#ifndef DET_ADV_THREADS
#define DET_ADV_THREADS 256
#endif
constexpr int ADV_THREADS = DET_ADV_THREADS;
constexpr int ADV_RPT = 2;
__global__ void __launch_bounds__(ADV_THREADS) k_advect_rows(Topo T, Bufs D, int gate) {
    const int b = blockIdx.y + D.b0;
    Carto* st = D.st + b;
    if (!gate_open(st, gate)) return;
    const int n = D.n;
    const size_t ub = (size_t)b * T.n_rows;
    float2* const pin = reinterpret_cast<float2*>(D.pos0) + ub;  // advected in place (see k_region)
    float2* const pout = pin;
    float2* __restrict__ pbest = reinterpret_cast<float2*>(D.best) + ub;
    const bool bestcopy = st->best_pending != 0;
    const float* uf = reinterpret_cast<const float*>(D.uf) + (size_t)b * D.nn * 2;
    const int v0 = blockIdx.x * (ADV_THREADS * ADV_RPT) + threadIdx.x;
    float2 p[ADV_RPT];
    TapF tp[ADV_RPT];
    Texels<float> tx[ADV_RPT];
#pragma unroll
    for (int q = 0; q < ADV_RPT; ++q) {
        const int v = v0 + q * ADV_THREADS;
        p[q] = v < T.n_rows ? pin[v] : make_float2(0.5f, 0.5f);
    }
#pragma unroll
    for (int q = 0; q < ADV_RPT; ++q) {
        tp[q] = field_tap_pf(n, p[q].x, p[q].y);
        tx[q] = field_load<float, TapF>(uf, tp[q]);
    }
    int ncl = 0;
#pragma unroll
    for (int q = 0; q < ADV_RPT; ++q) {
        const int v = v0 + q * ADV_THREADS;
        if (v >= T.n_rows) continue;
        const float2 s = field_blend_f(tx[q], tp[q]);
        const float mx = p[q].x + s.x, my = p[q].y + s.y;
        const float cx = mx < 0.0f ? 0.0f : (mx > 1.0f ? 1.0f : mx);  // np.clip (no NaNs here)
        const float cy = my < 0.0f ? 0.0f : (my > 1.0f ? 1.0f : my);
        ncl += (cx != mx) + (cy != my);
        pout[v] = make_float2(cx, cy);
        if (bestcopy) pbest[v] = p[q];
    }
    ncl = warp_sum(ncl);
    if ((threadIdx.x & 31) == 0 && ncl) atomicAdd(&st->clamps, (unsigned long long)ncl);
}

// Advect as its own flat kernel, float64 field and state (DET_SPLIT_ADVECT=1 on the float64 path):
// k_region's phase A arithmetic (displacement.py:209-238 op order) at full occupancy, ADV_RPT rows
// per thread; k_region then rasterises the rows written here (M_POSTADV).
__global__ void __launch_bounds__(ADV_THREADS) k_advect_rows64(Topo T, Bufs D, int gate) {
    const int b = blockIdx.y + D.b0;
    Carto* st = D.st + b;
    if (!gate_open(st, gate)) return;
    const int n = D.n;
    const size_t ub = (size_t)b * T.n_rows;
    double2* const pin = reinterpret_cast<double2*>(D.pos0) + ub;  // advected in place (see k_region)
    double2* __restrict__ pbest = reinterpret_cast<double2*>(D.best) + ub;
    const bool bestcopy = st->best_pending != 0;
    const double* uf = reinterpret_cast<const double*>(D.uf) + (size_t)b * D.nn * 2;
    const int v0 = blockIdx.x * (ADV_THREADS * ADV_RPT) + threadIdx.x;
    double2 p[ADV_RPT];
    Tap tp[ADV_RPT];
    Texels<double> tx[ADV_RPT];
#pragma unroll
    for (int q = 0; q < ADV_RPT; ++q) {
        const int v = v0 + q * ADV_THREADS;
        p[q] = v < T.n_rows ? pin[v] : make_double2(0.5, 0.5);
    }
#pragma unroll
    for (int q = 0; q < ADV_RPT; ++q) {
        tp[q] = field_tap(n, p[q].x, p[q].y);
        tx[q] = field_load<double, Tap>(uf, tp[q]);
    }
    int ncl = 0;
#pragma unroll
    for (int q = 0; q < ADV_RPT; ++q) {
        const int v = v0 + q * ADV_THREADS;
        if (v >= T.n_rows) continue;
        const double2 sm = field_blend<double, Tap>(tx[q], tp[q]);
        const double mx = p[q].x + sm.x, my = p[q].y + sm.y;
        const double cx = mx < 0.0 ? 0.0 : (mx > 1.0 ? 1.0 : mx);  // np.clip (no NaNs here)
        const double cy = my < 0.0 ? 0.0 : (my > 1.0 ? 1.0 : my);
        ncl += (cx != mx) + (cy != my);
        pin[v] = make_double2(cx, cy);
        if (bestcopy) pbest[v] = p[q];
    }
    ncl = warp_sum(ncl);
    if ((threadIdx.x & 31) == 0 && ncl) atomicAdd(&st->clamps, (unsigned long long)ncl);
}

// Advect once per UNIQUE vertex (float64 field and state): rows duplicating a shared vertex start
// bit-identical and evolve bit-identically (the update is a function of the position alone), so
// one thread advects the vertex from its first row and writes the result to every row of the
// vertex (CSR uq_off / uq_rows) -- half the taps and texel gathers of the per-row advect.  The
// clamp count is per row, as the reference counts it over the full vertex array
// (displacement.py:229-238): a vertex's clamped coordinates count once per row.
#ifndef DET_UQ_PER_THREAD
#define DET_UQ_PER_THREAD 1  // unique vertices per thread (1: 46.4k, 2: 46.0k, 4: 44.6k it/s)
#endif
constexpr int UQ_PT = DET_UQ_PER_THREAD;
__global__ void __launch_bounds__(ADV_THREADS) k_advect_uniq64(Topo T, Bufs D, int gate, const int* __restrict__ uq_row0,
                                                             const int* __restrict__ uq_off,
                                                             const int* __restrict__ uq_rows, int n_uniq) {
    const int b = blockIdx.y + D.b0;
    Carto* st = D.st + b;
    if (!gate_open(st, gate)) return;
    const int n = D.n;
    const size_t ub = (size_t)b * T.n_rows;
    double2* const pin = reinterpret_cast<double2*>(D.pos0) + ub;  // advected in place (see k_region)
    double2* __restrict__ pbest = reinterpret_cast<double2*>(D.best) + ub;
    const bool bestcopy = st->best_pending != 0;
    const double* uf = reinterpret_cast<const double*>(D.uf) + (size_t)b * D.nn * 2;
    const int u0 = blockIdx.x * (ADV_THREADS * UQ_PT) + threadIdx.x;
    int o[UQ_PT + 1 > 2 ? UQ_PT + 1 : 2][2];
    double2 p[UQ_PT];
    Tap tp[UQ_PT];
    Texels<double> tx[UQ_PT];
#pragma unroll
    for (int q = 0; q < UQ_PT; ++q) {
        const int u = u0 + q * ADV_THREADS;
        o[q][0] = u < n_uniq ? uq_off[u] : 0;
        o[q][1] = u < n_uniq ? uq_off[u + 1] : 0;
        p[q] = u < n_uniq ? pin[uq_row0[u]] : make_double2(0.5, 0.5);
    }
#pragma unroll
    for (int q = 0; q < UQ_PT; ++q) {
        tp[q] = field_tap(n, p[q].x, p[q].y);
        tx[q] = field_load<double, Tap>(uf, tp[q]);
    }
    int ncl = 0;
#pragma unroll
    for (int q = 0; q < UQ_PT; ++q) {
        const double2 sm = field_blend<double, Tap>(tx[q], tp[q]);
        const double mx = p[q].x + sm.x, my = p[q].y + sm.y;
        const double cx = mx < 0.0 ? 0.0 : (mx > 1.0 ? 1.0 : mx);  // np.clip (no NaNs here)
        const double cy = my < 0.0 ? 0.0 : (my > 1.0 ? 1.0 : my);
        const int o0 = o[q][0], o1 = o[q][1];
        ncl += ((cx != mx) + (cy != my)) * (o1 - o0);
        const double2 c = make_double2(cx, cy);
        for (int i = o0; i < o1; ++i) {
            const int v = uq_rows[i];
            pin[v] = c;
            if (bestcopy) pbest[v] = p[q];
        }
    }
    if (__any_sync(FULL, ncl != 0)) {  // clamping is rare (the map's border)
        ncl = warp_sum(ncl);
        if ((threadIdx.x & 31) == 0 && ncl) atomicAdd(&st->clamps, (unsigned long long)ncl);
    }
}

// Unique-vertex STATE (float64 graph iterations): inside a graph launch the cartogram's positions
// live in D.upos, one double2 per unique vertex -- k_uq_gather fills it from the rows at the
// launch's start, k_advect_uniq64s advects it in place (coalesced reads and writes, no row
// scatter), k_region<.., UQ> rasterises through Topo::row_uniq, and k_uq_expand writes the rows
// (and the best rows, when a best copy was taken) back at the launch's end.  Same arithmetic as
// k_advect_uniq64: bit-identical rows.
__global__ void __launch_bounds__(256) k_uq_gather(Topo T, Bufs D, int gate, const int* __restrict__ uq_row0) {
    const int b = blockIdx.y + D.b0;
    const bool open = gate_open(D.st + b, gate);
    if (blockIdx.x == 0 && threadIdx.x == 0) D.uq_flag[b] = open ? 2 : 0;
    if (!open) return;
    const double2* pin = reinterpret_cast<const double2*>(D.pos0) + (size_t)b * T.n_rows;
    double2* up = D.upos + (size_t)b * D.n_uniq;
    unsigned char* band0 = D.uq_band[0] ? D.uq_band[0] + (size_t)b * D.uq_bstride : nullptr;
    const int lgH = __ffs(D.H) - 1;
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < D.n_uniq; u += gridDim.x * blockDim.x) {
        const double2 p = pin[uq_row0[u]];
        up[u] = p;
        if (band0) band0[u] = tap_band(D.n, lgH, p.y);  // band-fused advect: the first iteration reads buffer 0
    }
}

__global__ void __launch_bounds__(256) k_uq_expand(Topo T, Bufs D) {
    const int b = blockIdx.y + D.b0;
    const int fl = D.uq_flag[b];
    if (!(fl & 2)) return;
    double2* pin = reinterpret_cast<double2*>(D.pos0) + (size_t)b * T.n_rows;
    double2* pbest = reinterpret_cast<double2*>(D.best) + (size_t)b * T.n_rows;
    const double2* up = D.upos + (size_t)b * D.n_uniq;
    const double2* ub = D.ubest + (size_t)b * D.n_uniq;
    const bool wb = (fl & 1) != 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < T.n_rows; v += gridDim.x * blockDim.x) {
        const int u = __ldg(T.row_uniq + v);
        pin[v] = up[u];
        if (wb) pbest[v] = ub[u];
    }
}

// One unique vertex advected in place on the unique-vertex state (the arithmetic of
// k_advect_uniq64s); COH: the field was written by this kernel (coherent loads).  Writes the
// vertex's band byte for the next iteration when bnext is given.  Returns its clamp count.
template <bool COH>
__device__ __forceinline__ int advect_uq_vertex(const Bufs& D, int n, int lgH, const double* uf, double2* up, double2* ub,
                                                bool bestcopy, const int* __restrict__ uq_off, unsigned char* bnext, int u) {
    const double2 p = up[u];
    const Tap tp = field_tap(n, p.x, p.y);
    const Texels<double> tx = COH ? field_load_coherent(uf, tp) : field_load<double, Tap>(uf, tp);
    const double2 sm = field_blend<double, Tap>(tx, tp);
    const double mx = p.x + sm.x, my = p.y + sm.y;
    const double cx = mx < 0.0 ? 0.0 : (mx > 1.0 ? 1.0 : mx);  // np.clip (no NaNs here)
    const double cy = my < 0.0 ? 0.0 : (my > 1.0 ? 1.0 : my);
    up[u] = make_double2(cx, cy);
    if (bestcopy) ub[u] = p;
    if (bnext) bnext[u] = tap_band(n, lgH, cy);
    const int nc = (cx != mx) + (cy != my);
    return nc ? nc * (uq_off[u + 1] - uq_off[u]) : 0;  // counted once per row (displacement.py:229-238)
}

// Band-fused advect, second part: the vertices whose tap straddles two bands (band byte 255), after
// k_sat3x<.., FA> advected all others from inside their band's sweep.
__global__ void __launch_bounds__(ADV_THREADS) k_advect_bnd(Topo T, Bufs D, int gate, const int* __restrict__ uq_off, int par) {
    const int b = blockIdx.y + D.b0;
    Carto* st = D.st + b;
    if (!gate_open(st, gate)) return;
    const int n = D.n, n_uniq = D.n_uniq;
    const bool bestcopy = st->best_pending != 0;
    const int u = blockIdx.x * ADV_THREADS + threadIdx.x;
    const unsigned char* bcur = D.uq_band[par] + (size_t)b * D.uq_bstride;
    int ncl = 0;
    if (u < n_uniq && bcur[u] == 255)
        ncl = advect_uq_vertex<false>(D, n, __ffs(D.H) - 1, reinterpret_cast<const double*>(D.uf) + (size_t)b * D.nn * 2,
                                      D.upos + (size_t)b * n_uniq, D.ubest + (size_t)b * n_uniq, bestcopy, uq_off,
                                      D.uq_band[par ^ 1] + (size_t)b * D.uq_bstride, u);
    if (bestcopy && blockIdx.x == 0 && threadIdx.x == 0) D.uq_flag[b] = 3;
    if (__any_sync(FULL, ncl != 0)) {
        ncl = warp_sum(ncl);
        if ((threadIdx.x & 31) == 0 && ncl) atomicAdd(&st->clamps, (unsigned long long)ncl);
    }
}

// Band-fused advect, first part (called by every warp of a k_sat3x<.., FA> CTA after the CTA's
// barrier at the end of its band sweep): scan the cartogram's band bytes for this band, compact the
// matching vertices into the warp's queue (512 ints of shared memory) and advect them 32 at a time
// while the band's field rows are still in L2 / L1.
__device__ __forceinline__ void advect_band_vertices(const Bufs& D, int b, int band, int par, int wl, int nwarps, int lane,
                                                     int* queue, const int* __restrict__ uq_off) {
    Carto* st = D.st + b;
    const int n = D.n, nU = D.n_uniq, lgH = __ffs(D.H) - 1;
    const bool bestcopy = st->best_pending != 0;
    const double* uf = reinterpret_cast<const double*>(D.uf) + (size_t)b * D.nn * 2;
    double2* up = D.upos + (size_t)b * nU;
    double2* ub = D.ubest + (size_t)b * nU;
    const unsigned char* bcur = D.uq_band[par] + (size_t)b * D.uq_bstride;
    unsigned char* bnext = D.uq_band[par ^ 1] + (size_t)b * D.uq_bstride;
    const unsigned pat = (unsigned)band * 0x01010101u;
    int qh = 0, qt = 0, ncl = 0;
    for (int base = wl * 256; base < nU; base += nwarps * 256) {
        const int u0 = base + lane * 8;
        uint2 w = make_uint2(0xFEFEFEFEu, 0xFEFEFEFEu);  // 254: no band
        if (u0 < D.uq_bstride) w = *reinterpret_cast<const uint2*>(bcur + u0);  // (pad bytes are 254)
        unsigned mlo = __vcmpeq4(w.x, pat), mhi = __vcmpeq4(w.y, pat);  // 0xFF per matching byte
        const int c = (__popc(mlo) + __popc(mhi)) >> 3;
        int tot;
        int pos = qt + warp_excl_scan_int(c, lane, &tot);
        while (mlo) {
            const int j = (__ffs(mlo) - 1) >> 3;
            mlo &= ~(0xFFu << (8 * j));
            queue[pos++ & 511] = u0 + j;
        }
        while (mhi) {
            const int j = (__ffs(mhi) - 1) >> 3;
            mhi &= ~(0xFFu << (8 * j));
            queue[pos++ & 511] = u0 + 4 + j;
        }
        qt += tot;
        __syncwarp();
        while (qt - qh >= 32) {
            ncl += advect_uq_vertex<true>(D, n, lgH, uf, up, ub, bestcopy, uq_off, bnext, queue[(qh + lane) & 511]);
            qh += 32;
        }
        __syncwarp();
    }
    if (lane < qt - qh)
        ncl += advect_uq_vertex<true>(D, n, lgH, uf, up, ub, bestcopy, uq_off, bnext, queue[(qh + lane) & 511]);
    if (__any_sync(FULL, ncl != 0)) {
        ncl = warp_sum(ncl);
        if (lane == 0 && ncl) atomicAdd(&st->clamps, (unsigned long long)ncl);
    }
}

__global__ void __launch_bounds__(ADV_THREADS) k_advect_uniq64s(Topo T, Bufs D, int gate, const int* __restrict__ uq_off) {
    const int b = blockIdx.y + D.b0;
    Carto* st = D.st + b;
    if (!gate_open(st, gate)) return;
    const int n = D.n, n_uniq = D.n_uniq;
    double2* const up = D.upos + (size_t)b * n_uniq;  // advected in place
    double2* __restrict__ ub = D.ubest + (size_t)b * n_uniq;
    const bool bestcopy = st->best_pending != 0;
    const double* uf = reinterpret_cast<const double*>(D.uf) + (size_t)b * D.nn * 2;
    const int u = blockIdx.x * ADV_THREADS + threadIdx.x;
    const bool in = u < n_uniq;
    const int o0 = in ? uq_off[u] : 0, o1 = in ? uq_off[u + 1] : 0;
    const double2 p = in ? up[u] : make_double2(0.5, 0.5);
    const Tap tp = field_tap(n, p.x, p.y);
    const Texels<double> tx = field_load<double, Tap>(uf, tp);
    const double2 sm = field_blend<double, Tap>(tx, tp);
    const double mx = p.x + sm.x, my = p.y + sm.y;
    const double cx = mx < 0.0 ? 0.0 : (mx > 1.0 ? 1.0 : mx);  // np.clip (no NaNs here)
    const double cy = my < 0.0 ? 0.0 : (my > 1.0 ? 1.0 : my);
    int ncl = ((cx != mx) + (cy != my)) * (o1 - o0);  // counted once per row (displacement.py:229-238)
    if (in) {
        up[u] = make_double2(cx, cy);
        if (bestcopy) ub[u] = p;
    }
    if (bestcopy && blockIdx.x == 0 && threadIdx.x == 0) D.uq_flag[b] = 3;
    if (__any_sync(FULL, ncl != 0)) {  // clamping is rare (the map's border)
        ncl = warp_sum(ncl);
        if ((threadIdx.x & 31) == 0 && ncl) atomicAdd(&st->clamps, (unsigned long long)ncl);
    }
}

#ifndef DET_ROW_RED
#define DET_ROW_RED 0  // 1: non-returning atomics + clash check + exact repaint (53.3k vs 54.7k: clashes are common)
#endif
#ifndef DET_ROW_TMA
#define DET_ROW_TMA 1
#endif
#ifndef DET_ROW_FILL16
#define DET_ROW_FILL16 0
#endif
#ifndef DET_ROW_PRE
#define DET_ROW_PRE 4
#endif
#ifndef DET_ROW_LONG
#define DET_ROW_LONG 24  // spans longer than this are painted by the whole warp, shorter ones by their own lane (8: 58.3k, 16: 61.4k, 24: 61.75k, 32: 61.45k, 48: 61.2k it/s)
#endif
constexpr int ROW_PRE = DET_ROW_PRE;  // span rounds k_row loads before it knows the row's count

// One warp per texture row; rpc rows per CTA.  ctrl_mode: -1 raster only (background
// count), 0 loop evaluation, 1 final re-evaluation.
__global__ void __launch_bounds__(256) k_row(Topo T, Bufs D, int gate, int ctrl_mode) {
    extern __shared__ uint32_t s_lab[];  // [rows per CTA][n]
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, rpc = blockDim.x >> 5;
    const int b = blockIdx.y + D.b0, n = D.n;
    const int j = blockIdx.x * rpc + wid;
    Carto* st = D.st + b;
    uint32_t* lab_s = s_lab + (size_t)wid * n;
    const size_t rb = (size_t)b * n + j;
    int* cnt = D.cnt_acc + (size_t)b * (T.R + 1);
    // the row's span count and its first ROW_PRE rounds of span slots are loaded together with
    // the gate word (cap >= 64), so the common row pays one memory round trip
    const unsigned long long* sp = D.spans + rb * D.cap;
    const int c0 = j < n ? D.rowcnt[rb] : 0;
    unsigned long long v_pre[ROW_PRE];
#pragma unroll
    for (int q = 0; q < ROW_PRE; ++q) v_pre[q] = (j < n && q * 32 + lane < D.cap) ? sp[q * 32 + lane] : 0ull;
    if (!gate_open(st, gate)) return;
    if (j < n) {
#if DET_ROW_FILL16
        for (int i = lane; i < (n >> 2); i += 32) reinterpret_cast<uint4*>(lab_s)[i] = make_uint4(SENT, SENT, SENT, SENT);
#else
        for (int i = lane; i < n; i += 32) lab_s[i] = SENT;  // (16-byte stores measured slower here)
#endif
        __syncwarp();
        if (lane == 0) {
            D.rowcnt[rb] = 0;
            if (c0 > D.cap) atomicOr(&st->err, (int)E_SPAN_OVF);
            if (c0 > 0) atomicMax(&D.maxspan[b], c0);
        }
        const int c = min(c0, D.cap);
        // slot s of the row's span list (prefetched rounds from registers)
        auto span_at = [&](int s0) -> unsigned long long {
            unsigned long long v = 0ull;
            if (s0 + lane < c) {
                if (s0 < ROW_PRE * 32) {  // a prefetched round (static register pick)
                    v = v_pre[0];
#pragma unroll
                    for (int q = 1; q < ROW_PRE; ++q)
                        if (s0 == q * 32) v = v_pre[q];
                } else {
                    v = sp[s0 + lane];
                }
            }
            return v;
        };
#if DET_ROW_RED
        // paint with non-returning shared atomicMin (no per-pixel wait on the old value); overlaps
        // are detected afterwards: the row's painted-pixel count equals the sum of its span lengths
        // unless two spans claimed a pixel
        int mylen = 0;
        for (int s0 = 0; s0 < c; s0 += 32) {
            const unsigned long long v = span_at(s0);
            const int lo = (int)(v & 0xFFFFull), hi = (int)((v >> 16) & 0xFFFFull);
            const uint32_t rk = (uint32_t)(v >> 32);
            const bool longspan = hi - lo > DET_ROW_LONG;
            mylen += hi - lo;
            if (!longspan)  // lane paints its own short span
                for (int i = lo; i < hi; ++i) atomicMin(&lab_s[i], rk);
            unsigned lm = __ballot_sync(FULL, longspan);
            while (lm) {  // the warp paints long spans together
                const int q = __ffs(lm) - 1;
                lm &= lm - 1;
                const int qlo = __shfl_sync(FULL, lo, q), qhi = __shfl_sync(FULL, hi, q);
                const uint32_t qrk = __shfl_sync(FULL, rk, q);
                for (int i = qlo + lane; i < qhi; i += 32) atomicMin(&lab_s[i], qrk);
            }
        }
        __syncwarp();
        // the label texture holds region RANKS (-1 = background); det_get_labels maps them
        // back to region indices (raster.py:107 stores indices) -- saves a gather per pixel
        int4* lab4 = reinterpret_cast<int4*>(D.labels + (size_t)b * D.nn + (size_t)j * n);
        const int4* src4 = reinterpret_cast<const int4*>(lab_s);
        int painted = 0;
        for (int i = lane; i < (n >> 2); i += 32) {
            const int4 x = src4[i];
            lab4[i] = x;  // SENT == -1 bitwise
            painted += (x.x != -1) + (x.y != -1) + (x.z != -1) + (x.w != -1);
        }
        // (warp_sum leaves the total in lane 0 only: broadcast, so the branch below is warp-uniform)
        const bool clash = __shfl_sync(FULL, warp_sum(painted) != warp_sum(mylen), 0);
        if (clash) {
            // a pixel was claimed twice on this row (spans of two regions, or of one region --
            // the original rule counts both): repaint the row with returning atomics, which
            // decrement the loser of every claim exactly as before (raster.py:142-146)
            for (int i = lane; i < n; i += 32) lab_s[i] = SENT;
            __syncwarp();
            for (int s0 = 0; s0 < c; s0 += 32) {
                const unsigned long long v = span_at(s0);
                const int lo = (int)(v & 0xFFFFull), hi = (int)((v >> 16) & 0xFFFFull);
                const uint32_t rk = (uint32_t)(v >> 32);
                for (int i = lo; i < hi; ++i) {
                    const uint32_t old = atomicMin(&lab_s[i], rk);
                    if (old != SENT) atomicAdd(&cnt[T.rank_region[max(old, rk)]], -1);
                }
            }
            __syncwarp();
            for (int i = lane; i < (n >> 2); i += 32) lab4[i] = src4[i];
            __threadfence();  // order the (rare) count corrections before this CTA signs off
        }
#else
        bool lost = false;
        for (int s0 = 0; s0 < c; s0 += 32) {
            const unsigned long long v = span_at(s0);
            const int lo = (int)(v & 0xFFFFull), hi = (int)((v >> 16) & 0xFFFFull);
            const uint32_t rk = (uint32_t)(v >> 32);
            const bool longspan = hi - lo > DET_ROW_LONG;
            if (!longspan) {  // lane paints its own short span, 4 claims in flight per step
                for (int i0 = lo; i0 < hi; i0 += 4) {
                    uint32_t old[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) old[q] = i0 + q < hi ? atomicMin(&lab_s[i0 + q], rk) : SENT;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (old[q] != SENT) {  // the higher rank loses the pixel
                            atomicAdd(&cnt[T.rank_region[max(old[q], rk)]], -1);
                            lost = true;
                        }
                    }
                }
            }
            unsigned lm = __ballot_sync(FULL, longspan);
            while (lm) {  // the warp paints long spans together
                const int q = __ffs(lm) - 1;
                lm &= lm - 1;
                const int qlo = __shfl_sync(FULL, lo, q), qhi = __shfl_sync(FULL, hi, q);
                const uint32_t qrk = __shfl_sync(FULL, rk, q);
                for (int i = qlo + lane; i < qhi; i += 32) {
                    const uint32_t old = atomicMin(&lab_s[i], qrk);
                    if (old != SENT) {
                        atomicAdd(&cnt[T.rank_region[max(old, qrk)]], -1);
                        lost = true;
                    }
                }
            }
        }
        __syncwarp();
        // the label texture holds region RANKS (-1 = background); det_get_labels maps them
        // back to region indices (raster.py:107 stores indices) -- saves a gather per pixel
        int* lab_g = D.labels + (size_t)b * D.nn + (size_t)j * n;
#if DET_ROW_TMA
        // the row leaves shared memory as one 1-D TMA bulk store issued by lane 0 (SENT == -1
        // bitwise); the generic-proxy paint is fenced for the async proxy first, and lane 0 waits
        // until the store has READ the shared row (wait_group.read) before the row can go away --
        // the global write itself completes asynchronously, before the grid does
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(lab_g),
                         "r"((unsigned)__cvta_generic_to_shared(lab_s)), "r"((unsigned)n * 4u)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        }
        __syncwarp();
#else
        int4* lab4 = reinterpret_cast<int4*>(lab_g);
        const int4* src4 = reinterpret_cast<const int4*>(lab_s);
        for (int i = lane; i < (n >> 2); i += 32) lab4[i] = src4[i];  // SENT == -1 bitwise
#endif
        if (lost) {  // order the (rare) count corrections before this CTA signs off
            __threadfence();
        }
#endif
    }
    if (ctrl_mode == CTRL_SEPARATE) return;  // the control step runs as k_ctrl after this kernel
    // ---- completion: the CTA that finishes the last row of this cartogram runs the control step ----
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&D.rowdone[b], 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) D.rowdone[b] = 0;
    ctrl_body(T, D, b, ctrl_mode);
}

// interpolate_vertices (temporal.py:293-302): out[f] = a + frac[f] * (b - a), same float64
// op order (no FMA); rows first, then the R statistics.
__global__ void k_interpolate(const double* __restrict__ a, const double* __restrict__ b, long long len,
                              const double* __restrict__ fr, int nf, double* __restrict__ out) {
    const long long total = len * nf;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(i / len);
        const long long e = i - (long long)f * len;
        out[i] = __dadd_rn(a[e], __dmul_rn(fr[f], __dsub_rn(b[e], a[e])));
    }
}

// Vertex-row format conversions of the float32-field path's float2 state (load: round to nearest;
// read-back: exact widening).
__global__ void k_rows_to_f32(const double2* __restrict__ in, long long len, float2* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
        const double2 p = in[i];
        out[i] = make_float2(__double2float_rn(p.x), __double2float_rn(p.y));
    }
}
__global__ void k_rows_to_f64(const float2* __restrict__ in, long long len, double2* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
        out[i] = to_d2(in[i]);
}

// Rank texture -> region-index texture (output format of rasterize_labels).
__global__ void k_rank_to_index(const int* __restrict__ rk, const int* __restrict__ rank_region, size_t nn,
                                int* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
        const int v = rk[i];
        out[i] = v < 0 ? -1 : rank_region[v];
    }
}

// Stage-level advect (displacement.py:229-238) on a float64 field.
__global__ void k_advect_points(const double* __restrict__ uf, int n, const double2* __restrict__ in, int np,
                                double2* __restrict__ out, unsigned long long* clamps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c = 0;
    if (i < np) {
        const double2 p = in[i];
        const double2 s = sample_field<double>(uf, n, p.x, p.y);
        const double mx = p.x + s.x, my = p.y + s.y;
        const double cx = fmin(fmax(mx, 0.0), 1.0), cy = fmin(fmax(my, 0.0), 1.0);
        c = (cx != mx) + (cy != my);
        out[i] = make_double2(cx, cy);
    }
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(clamps, c);
}

// Stage-level build_density (raster.py:166-184): histogram then gather.
__global__ void k_hist(const int* __restrict__ lab, size_t nn, int R, int* cnt) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
        const int L = lab[i];
        atomicAdd(&cnt[L < 0 ? R : L], 1);
    }
}
__global__ void k_density(const int* __restrict__ lab, size_t nn, int R, const double* __restrict__ stats,
                          const int* __restrict__ cnt, double bdv, double* d) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
        const int L = lab[i];
        d[i] = L < 0 ? bdv : stats[L] / (double)cnt[L];
    }
}

// Region.area(): signed shoelace over the region's rings (geomodel.py:24-31, 63-65),
// on the rows of the selected position buffer.
__global__ void k_areas(Topo T, const double2* __restrict__ rp, const int* __restrict__ ring_start,
                        const int* __restrict__ region_ring0, double* out) {
    __shared__ double s_red[33];
    const int r = blockIdx.x;
    double acc = 0.0;
    for (int q = region_ring0[r]; q < region_ring0[r + 1]; ++q) {
        const int a = ring_start[q], e = ring_start[q + 1];
        if (e - a < 3) continue;
        for (int v = a + threadIdx.x; v < e; v += blockDim.x) {
            const double2 p = rp[v], nx = rp[v + 1 < e ? v + 1 : a];
            acc += p.x * nx.y - nx.x * p.y;
        }
    }
    const double s = block_reduce<0, double>(acc, 0.0, s_red);
    if (threadIdx.x == 0) out[r] = 0.5 * s;
}

}  // namespace det
