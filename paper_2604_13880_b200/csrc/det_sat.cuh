// Straight + 45-degree-tilted integral images -> displacement field (sm_100a).
//
// Replaces integral.py:47-169 (straight_inims / tilted_inims) and
// displacement.py:102-131,198-206 (mapping_grid - base_mapping) with three
// band-parallel kernels that never materialise the eight channels:
//
//   rho(j,i) = m * d(j,i) / C - 1      (residual density; by linearity of every
//                                       channel, u = t(d) - t(const) equals the
//                                       anchor combination of rho's channels / 2m)
//   A(j,i)   = sum_{i'<=i} rho(j,i')   (row prefix, clamped: A(j,i>=n) = row total)
//
// Straight channels come from alpha(j,i) = sum_{j'<=j} A(j',i).  The tilted ones
// come from the rotated-lattice sums R(U,V) = sum_{i'+j'<=U, i'-j'<=V} rho, which
// split into an up-left diagonal prefix UL of A above the row and a down-left one
// DL at/below it:  R(U,V) = UL(j-1,i-1) + DL(j,i)  (U=i+j, V=i-j), and
//   left   beta_t  = R(U,V-1)              = UL(j,i-1)   + DL(j+1,i-1)
//   top    alpha_t = Tu(U-1) - R(U-1,V-1) + rho(j,i),   R(U-1,V-1) = UL(j-1,i-2) + DL(j,i-1)
//   bottom gamma_t = Tv(V) - R(U,V)
//   right  delta_t = C - alpha_t - beta_t - gamma_t
// with Tu/Tv the anti-diagonal / diagonal prefix totals.  This reproduces the
// reference's sector tie rule (integral.py:9-14, oracle tests/oracles.py:30-54).
//
// The texture is cut into bands of H rows (one CTA per band and cartogram):
//   k_sat1  per-band sums of rho along columns, diagonals and anti-diagonals
//           (streamed one row at a time, one barrier per row), x-prefixed once at
//           the band end, plus row totals;
//   k_sat2  band-direction exclusive prefixes / inclusive suffixes (the carries)
//           and image totals -- every value k_sat3 needs, ready to load;
//   k_sat3  per band: load the carries, then one top-down sweep computing A,
//           alpha, UL and the in-band up-right ray URin (DL = DLtot - URin), and
//           the displacement u at every pixel centre (or the 8 channels).
// In-band arithmetic follows the field mode: float64 for the float64 field (the default) and the
// stage-level channel dumps, float32 for the float32/mixed fields; band carries are float64 always.
#pragma once
#include <type_traits>
#include "det_common.cuh"

namespace det {

// Residual density of CPT consecutive pixels of row j in the accumulator type A
// (float32 in the float32-field mode, float64 otherwise).  `lut` is the cartogram's
// residual-density table (indexed by region rank, background at R): a shared-memory
// copy when it fits (LUTS), else global memory.
template <int CPT, int SRC, typename A, bool LUTS>
__device__ __forceinline__ void load_rho(const Bufs& D, const SatSrc& S, const A* lut, int R, int b, int j, int x0,
                                         A (&rho)[CPT]) {
    const int n = D.n;
    if (x0 >= n) {
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = (A)0;
        return;
    }
    if (SRC == SRC_LABELS) {
        const int* lab = D.labels + (size_t)b * D.nn + (size_t)j * n + x0;
        int L[CPT];
        if (CPT == 2) {
            const int2 v = *reinterpret_cast<const int2*>(lab);
            L[0] = v.x; L[1] = v.y;
        } else {
#pragma unroll
            for (int q = 0; q < CPT; q += 4) {
                const int4 v = *reinterpret_cast<const int4*>(lab + q);
                L[q] = v.x; L[q + 1] = v.y; L[q + 2] = v.z; L[q + 3] = v.w;
            }
        }
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int ix = L[k] < 0 ? R : L[k];
            rho[k] = LUTS ? lut[ix] : __ldg(lut + ix);
        }
    } else {
        const double* d = S.d + (size_t)b * D.nn + (size_t)j * n + x0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = (A)__dadd_rn(__dmul_rn(d[k], S.scale), S.offset);
    }
}

// The cartogram's LUT in the accumulator type: global pointer, copied to `s_lut` when LUTS.
// BIAS: the shared copy is stored background-first (s_lut[0] = background, s_lut[r+1] = rank r) and
// the returned pointer is s_lut + 1, so a label L >= -1 indexes it directly (no background select).
template <typename A, bool LUTS, bool BIAS = false>
__device__ __forceinline__ const A* band_lut(const Bufs& D, int R, int b, A* s_lut) {
    const A* g = sizeof(A) == 4 ? reinterpret_cast<const A*>(D.lutf + (size_t)b * (R + 1))
                                : reinterpret_cast<const A*>(D.lut + (size_t)b * (R + 1));
    if constexpr (!LUTS) {
        return g;
    } else if constexpr (BIAS) {
        for (int i = threadIdx.x; i <= R; i += blockDim.x) s_lut[i] = __ldg(g + (i == 0 ? R : i - 1));
        return s_lut + 1;  // published by the caller's first barrier
    } else {
        for (int i = threadIdx.x; i <= R; i += blockDim.x) s_lut[i] = __ldg(g + i);
        return s_lut;  // published by the caller's first barrier
    }
}

// shared-memory LUT length (entries), rounded so what follows stays 8-byte aligned
__host__ __device__ __forceinline__ int lut_smem_len(int R) { return (R + 2) & ~1; }

// Label rows staged through a KP-slot shared-memory ring with 1-D TMA bulk copies
// (cp.async.bulk, completion on one mbarrier per slot): one elected thread moves a whole row
// (n int32, 16-byte aligned) per copy, so no thread spends instructions or registers on the
// prefetch.  Row j sits in slot (j - jt) % KP.  At the start of iteration r the elected thread
// refills the slot every thread consumed in iteration r - 1 -- that iteration's __syncthreads
// has passed, and a proxy fence orders those generic reads before the async-proxy write --
// with row r + KP - 1, so the prefetch distance is KP - 1 rows.
// ring slots (prefetch distance KP - 1 rows): 4, or 2 for 8192-column rows, whose ring would
// not fit next to the carry windows in one CTA's shared memory
#ifndef DET_KP3
#define DET_KP3 4
#endif
__host__ __device__ constexpr int lab_kp(int cols) { return cols >= 8192 ? 2 : (cols >= 4096 ? 4 : DET_KP3); }
// k_sat1 takes each row one iteration early (its LUT gathers overlap the previous row), so it keeps
// a deeper ring where shared memory allows
#ifndef DET_KP1
#define DET_KP1 6
#endif
__host__ __device__ constexpr int lab_kp1(int cols) { return cols >= 8192 ? 2 : (cols >= 4096 ? 4 : DET_KP1); }

// k_sat3x: entries per phase of its phase-split carry windows for CTAs of NWC 128-column slices
// (compile-time: the band height is below the slice width)
__host__ __device__ constexpr int sat3x_phase_len(int NWC) { return (NWC * 128 + 128 + 6) / 4 + 2; }

// first 16-byte aligned int slot at or after p (cp.async 16-byte copies and int4 reads)
// (offset arithmetic on the pointer itself, so the compiler keeps it in the shared window: LDS,
// not generic LD, for the ring reads)
template <typename T>
__device__ __forceinline__ int* align16(T* p) {
    char* c = reinterpret_cast<char*>(p);
    const unsigned mis = (unsigned)(reinterpret_cast<uintptr_t>(c) & 15u);
    return reinterpret_cast<int*>(c + ((16u - mis) & 15u));
}

template <int CPT, int KP>
struct LabelRing {
    int* q;          // KP slots of `stride` ints
    uint64_t* bar;   // KP mbarriers
    const int* lab;  // cartogram's label texture, row 0
    int stride, n, x0, jt, j_last;
    bool active;
    __device__ __forceinline__ static unsigned sm(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
    // one thread, before the CTA's first barrier
    __device__ __forceinline__ void init() {
        if (threadIdx.x == 0) {
#pragma unroll
            for (int s = 0; s < KP; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm(bar + s)));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
    }
    __device__ __forceinline__ void issue(int row, int slot) {  // elected thread only
        if (row > j_last) return;
        const unsigned bytes = (unsigned)n * 4u;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm(bar + slot)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         sm(q + slot * stride)),
                     "l"(lab + (size_t)row * n), "r"(bytes), "r"(sm(bar + slot))
                     : "memory");
    }
    __device__ __forceinline__ void prologue() {  // after init() and a barrier
        if (threadIdx.x == 0) {
#pragma unroll
            for (int p = 0; p < KP - 1; ++p) issue(jt + p, p);
        }
    }
    __device__ __forceinline__ void wait(int slot, unsigned parity) {
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(sm(bar + slot)), "r"(parity)
                : "memory");
        }
    }
    // labels of row j -> residual densities (refilling the previous row's slot first)
    template <typename A, bool BIAS = false>
    __device__ __forceinline__ void take(int j, const A* lut, int R, A (&rho)[CPT]) {
        const int r = j - jt;
        if (threadIdx.x == 0) issue(j + KP - 1, (r + KP - 1) % KP);
        wait(r % KP, (unsigned)((r / KP) & 1));
        if (active) {
            const int* src = q + (r % KP) * stride + x0;
            int L[CPT];
            if (CPT % 4 == 0) {
#pragma unroll
                for (int c = 0; c < CPT; c += 4) {
                    const int4 v = *reinterpret_cast<const int4*>(src + c);
                    L[c] = v.x; L[c + 1] = v.y; L[c + 2] = v.z; L[c + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < CPT; c += 2) {
                    const int2 v = *reinterpret_cast<const int2*>(src + c);
                    L[c] = v.x; L[c + 1] = v.y;
                }
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = BIAS ? lut[L[k]] : lut[L[k] < 0 ? R : L[k]];
        } else {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = (A)0;
        }
    }
};

// 256-bit global stores (sm_100: STG.256): one whole 32-byte sector per thread and instruction
__device__ __forceinline__ void st_global_v4f64(void* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void st_global_v8f32(void* p, float a, float b, float c, float d, float e, float f,
                                                float g, float h) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d), "f"(e), "f"(f), "f"(g), "f"(h)
                 : "memory");
}

template <typename A>
__device__ __forceinline__ A warp_incl_scan_t(A v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const A t = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// In-place inclusive prefix of a[0..len) in shared memory by the whole CTA (float64 carry).
template <typename A>
__device__ void block_prefix_smem(A* a, double* out, int len, double* sm) {
    const int nt = blockDim.x;
    const int per = (len + nt - 1) / nt;
    const int s = min(len, threadIdx.x * per), e = min(len, s + per);
    double loc = 0.0;
    for (int i = s; i < e; ++i) loc += (double)a[i];
    double tot;
    double run = block_excl_scan(loc, sm, &tot);
    for (int i = s; i < e; ++i) {
        run += (double)a[i];
        out[i] = run;
    }
}

// ---------------------------------------------------------------------------------
// Per-band sums, x-prefixed:  CS_b(x) = sum_{j in band, i<=x} rho,
// DG_b(v) = sum_{j in band, i-j<=v} rho (compact index q = v + jb, q in [0, n+H-1)),
// AD_b(w) = sum_{j in band, i+j<=w} rho (compact index q = w - jt).  Outside the
// compact range the prefixes are 0 (below) or the band total (above).  In-band sums
// in A; the x-prefixes and everything downstream in float64.
template <int CPT, int NT, int SRC, typename A, bool LUTS>
__global__ void __launch_bounds__(NT) k_sat1(Topo T, Bufs D, SatSrc S, int gate) {
    extern __shared__ unsigned char s_raw1[];  // dg[L] | ad[L] | lut (LUTS) | row partials [H][NW], all in A
    constexpr int NW = NT / 32;
    __shared__ A s_bd[3][32];
    __shared__ A s_ba[3][32];
    __shared__ double s_red[33];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, L = n + H - 1, R = T.R;
    const int x0 = t * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    A* dg = reinterpret_cast<A*>(s_raw1);
    A* ad = dg + L;
    A* s_lut = ad + L;
    A* s_rows = s_lut + (LUTS ? lut_smem_len(R) : 0);
    const A* lut = band_lut<A, LUTS>(D, R, b, s_lut);
    if (LUTS) __syncthreads();
    // labels through the shared-memory ring on the float path (the float64 path's carry windows
    // leave no room for it at 8192 columns); register prefetch otherwise
    constexpr bool RING = SRC == SRC_LABELS && sizeof(A) == 4;
    __shared__ uint64_t s_bar[6];
    LabelRing<CPT, lab_kp1(CPT * NT)> ring;
    if (RING) {
        ring.q = align16(s_rows + H * NW);
        ring.bar = s_bar;
        ring.lab = D.labels + (size_t)b * D.nn;
        ring.stride = NT * CPT;
        ring.n = n;
        ring.x0 = x0;
        ring.jt = jt;
        ring.j_last = jb;
        ring.active = x0 < n;
        ring.init();
        __syncthreads();
        ring.prologue();
    }
    A cs[CPT], pd[CPT], pa[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) cs[k] = pd[k] = pa[k] = (A)0;

    // densities one row ahead: row j+1's label wait and LUT gathers are issued before row j's work
    A rho_n[CPT];
    if (RING) ring.take(jt, lut, R, rho_n);
    else load_rho<CPT, SRC, A, LUTS>(D, S, lut, R, b, jt, x0, rho_n);
    int slot = 0, ps = 2;  // rotating boundary slots: (j - jt) % 3, (j - jt + 2) % 3
    for (int j = jt; j <= jb; ++j) {
        A rho[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
        if (j < jb) {
            if (RING) ring.take(j + 1, lut, R, rho_n);  // refills row j's slot: every take(j) preceded barrier j-1
            else load_rho<CPT, SRC, A, LUTS>(D, S, lut, R, b, j + 1, x0, rho_n);
        }
        A ts = (A)0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) ts += rho[k];
        ts = warp_sum(ts);
        if (lane == 0) s_rows[(j - jt) * NW + w] = ts;  // row totals are summed after the sweep
        __syncthreads();
        A left = __shfl_up_sync(FULL, pd[CPT - 1], 1);
        A right = __shfl_down_sync(FULL, pa[0], 1);
        if (lane == 0) left = (w == 0 || j == jt) ? (A)0 : s_bd[ps][w - 1];
        if (lane == 31) right = (w == NW - 1 || j == jt) ? (A)0 : s_ba[ps][w + 1];
        A nd_[CPT], na_[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            nd_[k] = rho[k] + (k == 0 ? left : pd[k - 1]);
            na_[k] = rho[k] + (k == CPT - 1 ? right : pa[k + 1]);
            cs[k] += rho[k];
        }
        if (j < jb) {
            // diagonal leaves the right edge: n is a multiple of CPT, so column n-1 is the last
            // column of thread n/CPT - 1 (a static register index -- no local-memory array)
            if (x0 == n - CPT) dg[n - 1 - j + jb] = nd_[CPT - 1];
            if (x0 == 0) ad[j - jt] = na_[0];                                           // anti-diagonal leaves left edge
        }
        if (lane == 31) s_bd[slot][w] = nd_[CPT - 1];
        if (lane == 0) s_ba[slot][w] = na_[0];
#pragma unroll
        for (int k = 0; k < CPT; ++k) { pd[k] = nd_[k]; pa[k] = na_[k]; }
        ps = slot;
        slot = slot == 2 ? 0 : slot + 1;
    }
    // band bottom: remaining diagonals / anti-diagonals end here; column sums -> x-prefix
    double csum = 0.0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        if (x < n) {
            dg[x] = pd[k];
            ad[jb - jt + x] = pa[k];
        }
        csum += x < n ? (double)cs[k] : 0.0;
    }
    double tot;
    double run = block_excl_scan(csum, s_red, &tot);  // (its barriers also publish dg/ad and s_rows)
    if (t < H) {  // row totals in float64, warp order (as the sweep produced them)
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) s += (double)s_rows[t * NW + q];
        D.rt[(size_t)b * n + jt + t] = s;
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        run += (double)cs[k];
        if (x < n) D.cs[bb * n + x] = run;
    }
    block_prefix_smem<A>(dg, D.dgc + bb * L, L, s_red);
    block_prefix_smem<A>(ad, D.adc + bb * L, L, s_red);
}

// ---------------------------------------------------------------------------------
// k_sat1w: k_sat1 for the float32 field with no CTA barrier in the row sweep.  Each warp owns a
// 32*CPT-column slice: it streams its slice of every label row through its own 1-D TMA ring and
// carries diagonal / anti-diagonal partial sums only inside the slice (zero at the slice edge).
// The partial leaving the slice after each row is recorded (exitD / exitA); a band is at most
// 64 rows <= the slice width, so a diagonal crosses at most one slice edge and its band sum is
// the recorded partial plus the neighbour slice's continuation, added once at the band end.
// Outputs equal k_sat1's (the in-band sums are grouped per slice).
template <int CPT, int KP>
struct WarpRing {
    int* q;          // KP slots of 32*CPT ints (this warp's)
    uint64_t* bar;   // KP mbarriers (this warp's)
    const int* lab;  // label row 0, this warp's first column
    int n, jt, j_last;
    unsigned bytes;  // valid bytes of the slice (0: slice beyond the texture)
    __device__ __forceinline__ static unsigned sm(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
    __device__ __forceinline__ void init(int lane) {
        if (lane == 0) {
#pragma unroll
            for (int s = 0; s < KP; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sm(bar + s)));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncwarp();
    }
    __device__ __forceinline__ void issue(int row, int slot) {  // lane 0 only
        if (row > j_last || bytes == 0) return;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sm(bar + slot)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         sm(q + slot * 32 * CPT)),
                     "l"(lab + (size_t)row * n), "r"(bytes), "r"(sm(bar + slot))
                     : "memory");
    }
    __device__ __forceinline__ void prologue(int lane) {
        if (lane == 0) {
#pragma unroll
            for (int p = 0; p < KP - 1; ++p) issue(jt + p, p);
        }
    }
    // row j -> residual densities; refills row j-1's slot (every lane finished reading it: the
    // __syncwarp below orders those reads before lane 0's async-proxy write)
    template <typename A, bool BIAS = false>
    __device__ __forceinline__ void take(int j, int lane, bool active, const A* lut, int R, A (&rho)[CPT]) {
        const int r = j - jt;
        __syncwarp();
        if (lane == 0) issue(j + KP - 1, (r + KP - 1) % KP);
        if (bytes == 0) {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = (A)0;
            return;
        }
        const int slot = r % KP;
        const unsigned parity = (unsigned)((r / KP) & 1);
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(sm(bar + slot)), "r"(parity)
                : "memory");
        }
        if (active) {
            const int* src = q + slot * 32 * CPT + lane * CPT;
            int L[CPT];
            if constexpr (CPT % 4 == 0) {
#pragma unroll
                for (int c = 0; c < CPT; c += 4) {
                    const int4 v = *reinterpret_cast<const int4*>(src + c);
                    L[c] = v.x; L[c + 1] = v.y; L[c + 2] = v.z; L[c + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < CPT; c += 2) {
                    const int2 v = *reinterpret_cast<const int2*>(src + c);
                    L[c] = v.x; L[c + 1] = v.y;
                }
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = BIAS ? lut[L[k]] : lut[L[k] < 0 ? R : L[k]];
        } else {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = (A)0;
        }
    }
};

#ifndef DET_SAT1W_LUTS
#define DET_SAT1W_LUTS 1
#endif
#ifndef DET_SAT1W_CPT
#define DET_SAT1W_CPT 4  // columns per thread of k_sat1w at CPT=4 configs (2: 49.7k, 4: 52.6k it/s)
#endif
//
// TAB (float64 field, for k_sat3w): also record, per band row r and slice w, the slice table
//   tab[0][w][r] = off(r, w): the row prefix left of the slice, sum_{w' < w} slice total(r, w')
//   tab[1][w][r] = E1(r, w):  sum over the slice of the diagonal partials pd(jt + r, .)
//   tab[2][w][r] = pd at the slice's last column, tab[3][w][r] = pa at its first column
// (D.tab + band * 4 * NW * H), from which k_sat3w's warps form every value crossing a slice edge.
template <int CPT, int NT, bool LUTS, typename A = float, bool TAB = false>
__global__ void __launch_bounds__(NT) k_sat1w(Topo T, Bufs D, int gate) {
    constexpr int NW = NT / 32, W = 32 * CPT, KP = lab_kp1(CPT * NT);
    // dg[L] | ad[L] | row partials [H][NW] | exitD [NW][H] | exitA [NW][H] | (TAB) E1 [NW][H] | rings (16-B aligned)
    extern __shared__ unsigned char s_raw1[];
    __shared__ uint64_t s_bar[NW * KP];
    __shared__ double s_red[33];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, L = n + H - 1, R = T.R;
    const int x0 = t * CPT, c0 = w * W;
    const bool active = x0 < n;
    const size_t bb = (size_t)b * D.nb + band;
    A* dg = reinterpret_cast<A*>(s_raw1);
    A* ad = dg + L;
    A* s_rows = ad + L;
    A* exD = s_rows + H * NW;
    A* exA = exD + NW * H;
    A* exE = exA + NW * H;  // TAB only
    const A* glut = sizeof(A) == 4 ? reinterpret_cast<const A*>(D.lutf + (size_t)b * (R + 1))
                                   : reinterpret_cast<const A*>(D.lut + (size_t)b * (R + 1));
    // LUTS: the LUT staged in shared memory after the rings
    A* ring_base = exA + NW * H * (TAB ? 2 : 1);
    A* s_lut = reinterpret_cast<A*>(align16(ring_base) + NW * KP * W);
    if (LUTS)  // background-first (see band_lut): labels index s_lut + 1 directly
        for (int i = t; i <= R; i += NT) s_lut[i] = __ldg(glut + (i == 0 ? R : i - 1));
    const A* lut = LUTS ? s_lut + 1 : glut;
    WarpRing<CPT, KP> ring;
    ring.q = align16(ring_base) + w * KP * W;
    ring.bar = s_bar + w * KP;
    ring.lab = D.labels + (size_t)b * D.nn + c0;
    ring.n = n;
    ring.jt = jt;
    ring.j_last = jb;
    ring.bytes = (unsigned)(max(0, min(W, n - c0)) * 4);
    ring.init(lane);
    ring.prologue(lane);
    if (LUTS) __syncthreads();  // LUT published

    A cs[CPT], pd[CPT], pa[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) cs[k] = pd[k] = pa[k] = (A)0;
    A rho_n[CPT];
    A ts_even = (A)0;  // the even row's partial, reduced together with the odd row (H is even)
    A ps_even = (A)0;  // TAB: the even row's diagonal-partial sum
    ring.template take<A, LUTS>(jt, lane, active, lut, R, rho_n);
    for (int j = jt; j <= jb; ++j) {
        A rho[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
        if (j < jb) ring.template take<A, LUTS>(j + 1, lane, active, lut, R, rho_n);  // next row's gathers in flight
        A ts = (A)0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) ts += rho[k];
        // slice row totals, two rows per butterfly: after one exchange the lower half-warp holds
        // the even row's partials and the upper half the odd row's, so 5 shuffles serve 2 rows
        if (TAB) {
        } else if (((j - jt) & 1) == 0) {
            ts_even = ts;
            if (j == jb) {  // odd band height (H = 1): the last row is reduced alone
                const A t1 = warp_sum(ts);
                if (lane == 0) s_rows[(j - jt) * NW + w] = t1;
            }
        } else {
            const bool up = (lane & 16) != 0;
            A keep = (up ? ts : ts_even) + __shfl_xor_sync(FULL, up ? ts_even : ts, 16);
#pragma unroll
            for (int o = 8; o; o >>= 1) keep += __shfl_xor_sync(FULL, keep, o);
            if (lane == 0) s_rows[(j - 1 - jt) * NW + w] = keep;
            if (lane == 16) s_rows[(j - jt) * NW + w] = keep;
        }
        A left = __shfl_up_sync(FULL, pd[CPT - 1], 1);
        A right = __shfl_down_sync(FULL, pa[0], 1);
        if (lane == 0) left = (A)0;    // partials restart at the slice edge
        if (lane == 31) right = (A)0;
        // in place, so the diagonal recurrence runs right to left and the anti-diagonal one left to
        // right (each reads its neighbour's previous-row partial before it is overwritten)
#pragma unroll
        for (int k = CPT - 1; k >= 0; --k) pd[k] = rho[k] + (k == 0 ? left : pd[k - 1]);
#pragma unroll
        for (int k = 0; k < CPT; ++k) pa[k] = rho[k] + (k == CPT - 1 ? right : pa[k + 1]);
#pragma unroll
        for (int k = 0; k < CPT; ++k) cs[k] += rho[k];
        if (lane == 31) exD[w * H + (j - jt)] = pd[CPT - 1];  // diagonal leaving the slice's right edge
        if (lane == 0) exA[w * H + (j - jt)] = pa[0];  // anti-diagonal leaving the slice's left edge
        if constexpr (TAB) {
            // slice row total and E1 (the slice's sum of this row's diagonal partials), two rows per
            // butterfly: the half-warps take the even / odd row, then the quarter-warps the total /
            // E1, so 6 shuffles serve 4 sums (lanes 0, 8, 16, 24 end with them)
            A ps = (A)0;
#pragma unroll
            for (int k = 0; k < CPT; ++k) ps += pd[k];
            const int r = j - jt;
            if ((r & 1) == 0 && j < jb) {
                ts_even = ts;
                ps_even = ps;
            } else {
                const bool odd = (r & 1) != 0;
                const bool up = (lane & 16) != 0, qp = (lane & 8) != 0;
                A kt, kp;
                if (odd) {
                    kt = (up ? ts : ts_even) + __shfl_xor_sync(FULL, up ? ts_even : ts, 16);
                    kp = (up ? ps : ps_even) + __shfl_xor_sync(FULL, up ? ps_even : ps, 16);
                } else {  // odd band height: the last row alone (both half-warps hold it)
                    kt = ts + __shfl_xor_sync(FULL, ts, 16);
                    kp = ps + __shfl_xor_sync(FULL, ps, 16);
                }
                A v = (qp ? kp : kt) + __shfl_xor_sync(FULL, qp ? kt : kp, 8);
#pragma unroll
                for (int o = 4; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
                const int r0 = odd ? r - 1 : r;
                if (lane == 0) s_rows[r0 * NW + w] = v;
                if (lane == 8) exE[w * H + r0] = v;
                if (odd && lane == 16) s_rows[r * NW + w] = v;
                if (odd && lane == 24) exE[w * H + r] = v;
            }
        }
    }
    __syncthreads();  // exits, row partials published
    // band-bottom entries + the neighbour slice's part of each crossing diagonal
    double csum = 0.0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        if (x < n) {
            const int xi = x - c0;                       // column inside the slice
            A vd = pd[k], va = pa[k];
            if (w > 0 && xi <= H - 2) vd += exD[(w - 1) * H + (H - 2 - xi)];
            const int xr = W - 1 - xi;                   // columns to the slice's right edge
            if (w < NW - 1 && c0 + W < n && xr <= H - 2) va += exA[(w + 1) * H + (H - 2 - xr)];
            dg[x] = vd;
            ad[H - 1 + x] = va;
        }
        csum += x < n ? (double)cs[k] : 0.0;
    }
    // diagonals leaving the texture's right edge / anti-diagonals leaving its left edge (j < jb)
    if (t < H - 1) {
        const int wl = (n - 1) / W;  // slice holding column n-1
        dg[n - 1 - (jt + t) + jb] = exD[wl * H + t];
        ad[t] = exA[t];
    }
    double tot;
    double run = block_excl_scan(csum, s_red, &tot);  // (its barriers also publish dg/ad)
    if (t < H) {  // row totals in float64, warp order
        double s = 0.0;
        double* tab = TAB ? D.tab + bb * 4 * NW * H : nullptr;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            if (TAB) tab[q * H + t] = s;  // off(t, q): the slice totals left of slice q
            s += (double)s_rows[t * NW + q];
        }
        D.rt[(size_t)b * n + jt + t] = s;
    }
    if constexpr (TAB) {
        double* tab = D.tab + bb * 4 * NW * H;
        for (int i = t; i < NW * H; i += NT) {
            tab[NW * H + i] = (double)exE[i];
            tab[2 * NW * H + i] = (double)exD[i];
            tab[3 * NW * H + i] = (double)exA[i];
        }
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        run += (double)cs[k];
        if (x < n) D.cs[bb * n + x] = run;
    }
    block_prefix_smem<A>(dg, D.dgc + bb * L, L, s_red);
    block_prefix_smem<A>(ad, D.adc + bb * L, L, s_red);
}

// ---------------------------------------------------------------------------------
// Band-direction carries.  Lanes: [0,n) columns x, [n,3n-1) diagonals (idx=v+n-1),
// [3n-1,5n-2) anti-diagonals w.  blockDim = 32*G (G band groups).  The last block
// column computes rowfull (row-total prefix) instead.  Outputs per band b:
//   csX[b][x]   = sum_{b'<b} CS_b'(x)                 (alpha carry)
//   dgXc[b][x]  = sum_{b'<b} DG_b'(x - jt + 1)        (UL carry, x in [0,n))
//   adSc[b][q]  = sum_{b'>=b} AD_b'(jt - 1 + q)        (DLtot window, q in [0,n+H))
// and totals csT[x] = colfull(x+1), dgT[idx] = Tv(v), adT[w] = Tu(w).
constexpr int SAT2_THREADS = 128;
constexpr int SAT2_CHUNK = 16;  // bands loaded per round (independent loads in flight)

__global__ void __launch_bounds__(SAT2_THREADS) k_sat2(Bufs D, int gate) {
    __shared__ double s_red[33];
    const int b = blockIdx.y + D.b0, t = threadIdx.x;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, nb = D.nb, L = n + H - 1, M = 2 * n - 1;
    if (blockIdx.x == gridDim.x - 1) {
        // rowfull[J] = sum_{j<J} rt[j]
        const double* rt = D.rt + (size_t)b * n;
        double* rf = D.rowfull + (size_t)b * (n + 1);
        const int per = (n + blockDim.x - 1) / blockDim.x;
        const int a = min(n, t * per), e = min(n, a + per);
        double s = 0.0;
        for (int i = a; i < e; ++i) s += rt[i];
        double tot;
        double run = block_excl_scan(s, s_red, &tot);
        for (int i = a; i < e; ++i) { rf[i] = run; run += rt[i]; }
        if (t == 0) rf[n] = tot;
        return;
    }
    // one thread per lane: every band of one column / diagonal / anti-diagonal, streamed in
    // chunks of independent loads (forward for the prefixes, backward for the suffix)
    const int lanes = n + 2 * M;
    const int l = blockIdx.x * blockDim.x + t;
    if (l >= lanes) return;
    const int type = l < n ? 0 : (l < n + M ? 1 : 2);
    const int idx = type == 0 ? l : (type == 1 ? l - n : l - n - M);
    const size_t base = (size_t)b * nb;
    auto val = [&](int band) -> double {
        if (type == 0) return D.cs[(base + band) * n + idx];
        const int q = type == 1 ? idx - (n - 1) + (band * H + H - 1)  // v + jb
                                : idx - band * H;                     // w - jt
        if (q < 0) return 0.0;
        return (type == 1 ? D.dgc : D.adc)[(base + band) * L + min(q, L - 1)];
    };
    double run = 0.0;
    if (type != 2) {
        for (int b0 = 0; b0 < nb; b0 += SAT2_CHUNK) {
            double v[SAT2_CHUNK];
#pragma unroll
            for (int k = 0; k < SAT2_CHUNK; ++k) v[k] = b0 + k < nb ? val(b0 + k) : 0.0;
#pragma unroll
            for (int k = 0; k < SAT2_CHUNK; ++k) {
                const int band = b0 + k;
                if (band >= nb) break;
                if (type == 0) {
                    D.csX[(base + band) * n + idx] = run;
                } else {
                    const int x = idx - n + band * H;  // v + jt - 1, v = idx - (n-1)
                    if (x >= 0 && x < n) D.dgXc[(base + band) * n + x] = run;
                }
                run += v[k];
            }
        }
        if (type == 0) D.csT[(size_t)b * n + idx] = run;
        else D.dgT[(size_t)b * M + idx] = run;
    } else {
        for (int e0 = nb; e0 > 0; e0 -= SAT2_CHUNK) {
            double v[SAT2_CHUNK];
#pragma unroll
            for (int k = 0; k < SAT2_CHUNK; ++k) v[k] = e0 - 1 - k >= 0 ? val(e0 - 1 - k) : 0.0;
#pragma unroll
            for (int k = 0; k < SAT2_CHUNK; ++k) {
                const int band = e0 - 1 - k;
                if (band < 0) break;
                run += v[k];
                const int q = idx - band * H + 1;  // w - (jt - 1)
                if (q >= 0 && q < L + 1) D.adSc[(base + band) * (L + 1) + q] = run;
            }
        }
        D.adT[(size_t)b * M + idx] = run;
    }
}

// Float32-field variant of k_sat2: each lane's bands are split over SAT2_PARTS warps of the CTA
// (one warp per part, 32 lanes per CTA), so every thread keeps at most SAT2P_CH band values in
// flight and the lane's bands are fetched in one memory round trip; the parts' sums are combined
// through shared memory.  Same outputs as k_sat2 (summation grouped by part).
#ifndef DET_SAT2_PARTS
#define DET_SAT2_PARTS 4
#endif
constexpr int SAT2_PARTS = DET_SAT2_PARTS;
constexpr int SAT2P_CH = 32 / DET_SAT2_PARTS;  // bands per part in registers (32 bands at 1024^2)

__global__ void __launch_bounds__(32 * SAT2_PARTS) k_sat2p(Bufs D, int gate) {
    __shared__ double s_part[SAT2_PARTS][32];
    __shared__ double s_red[33];
    const int b = blockIdx.y + D.b0, t = threadIdx.x, lane = t & 31, part = t >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, nb = D.nb, L = n + H - 1, M = 2 * n - 1;
    if (blockIdx.x == gridDim.x - 1) {
        // rowfull[J] = sum_{j<J} rt[j]
        const double* rt = D.rt + (size_t)b * n;
        double* rf = D.rowfull + (size_t)b * (n + 1);
        const int per = (n + blockDim.x - 1) / blockDim.x;
        const int a = min(n, t * per), e = min(n, a + per);
        double s = 0.0;
        for (int i = a; i < e; ++i) s += rt[i];
        double tot;
        double run = block_excl_scan(s, s_red, &tot);
        for (int i = a; i < e; ++i) { rf[i] = run; run += rt[i]; }
        if (t == 0) rf[n] = tot;
        return;
    }
    const int lanes = n + 2 * M;
    const int l = blockIdx.x * 32 + lane;
    const bool ok = l < lanes;
    const int type = l < n ? 0 : (l < n + M ? 1 : 2);
    const int idx = type == 0 ? l : (type == 1 ? l - n : l - n - M);
    const size_t base = (size_t)b * nb;
    auto val = [&](int band) -> double {
        if (type == 0) return D.cs[(base + band) * n + idx];
        const int q = type == 1 ? idx - (n - 1) + (band * H + H - 1)  // v + jb
                                : idx - band * H;                     // w - jt
        if (q < 0) return 0.0;
        return (type == 1 ? D.dgc : D.adc)[(base + band) * L + min(q, L - 1)];
    };
    const int per = (nb + SAT2_PARTS - 1) / SAT2_PARTS;
    const int p0 = min(nb, part * per), p1 = min(nb, p0 + per);
    // pass 1: this part's sum (the first chunk stays in registers for pass 2)
    double v0[SAT2P_CH];
    double loc = 0.0;
#pragma unroll
    for (int k = 0; k < SAT2P_CH; ++k) {
        v0[k] = (ok && p0 + k < p1) ? val(p0 + k) : 0.0;
        loc += v0[k];
    }
    // (more bands per part than the register chunk -- short bands, few frames: later chunks are loaded
    // SAT2P_CH at a time, so their round trips overlap instead of running one band after another)
    for (int c0 = p0 + SAT2P_CH; c0 < p1; c0 += SAT2P_CH) {
        double v[SAT2P_CH];
#pragma unroll
        for (int k = 0; k < SAT2P_CH; ++k) v[k] = (ok && c0 + k < p1) ? val(c0 + k) : 0.0;
#pragma unroll
        for (int k = 0; k < SAT2P_CH; ++k) loc += v[k];
    }
    s_part[part][lane] = loc;
    __syncthreads();
    if (!ok) return;
    double run = 0.0;  // forward: parts before this one; backward (type 2): parts after it
    if (type != 2) {
        for (int q = 0; q < part; ++q) run += s_part[q][lane];
        auto put = [&](int band) {
            if (type == 0) {
                D.csX[(base + band) * n + idx] = run;
            } else {
                const int x = idx - n + band * H;  // v + jt - 1, v = idx - (n-1)
                if (x >= 0 && x < n) D.dgXc[(base + band) * n + x] = run;
            }
        };
#pragma unroll
        for (int k = 0; k < SAT2P_CH; ++k) {
            if (p0 + k < p1) {
                put(p0 + k);
                run += v0[k];
            }
        }
        for (int c0 = p0 + SAT2P_CH; c0 < p1; c0 += SAT2P_CH) {
            double v[SAT2P_CH];
#pragma unroll
            for (int k = 0; k < SAT2P_CH; ++k) v[k] = c0 + k < p1 ? val(c0 + k) : 0.0;
#pragma unroll
            for (int k = 0; k < SAT2P_CH; ++k) {
                if (c0 + k < p1) {
                    put(c0 + k);
                    run += v[k];
                }
            }
        }
        if (part == SAT2_PARTS - 1) {
            if (type == 0) D.csT[(size_t)b * n + idx] = run;
            else D.dgT[(size_t)b * M + idx] = run;
        }
    } else {
        for (int q = SAT2_PARTS - 1; q > part; --q) run += s_part[q][lane];
        auto put = [&](int band) {
            const int q = idx - band * H + 1;  // w - (jt - 1)
            if (q >= 0 && q < L + 1) D.adSc[(base + band) * (L + 1) + q] = run;
        };
        for (int c1 = p1; c1 > p0 + SAT2P_CH; c1 -= SAT2P_CH) {  // bands c1-1 down to max(c1 - CH, p0 + CH)
            double v[SAT2P_CH];
#pragma unroll
            for (int k = 0; k < SAT2P_CH; ++k) v[k] = c1 - 1 - k >= p0 + SAT2P_CH ? val(c1 - 1 - k) : 0.0;
#pragma unroll
            for (int k = 0; k < SAT2P_CH; ++k) {
                if (c1 - 1 - k >= p0 + SAT2P_CH) {
                    run += v[k];
                    put(c1 - 1 - k);
                }
            }
        }
#pragma unroll
        for (int k = SAT2P_CH - 1; k >= 0; --k) {
            if (p0 + k < p1) {
                run += v0[k];
                put(p0 + k);
            }
        }
        if (part == 0) D.adT[(size_t)b * M + idx] = run;
    }
}

// ---------------------------------------------------------------------------------
// Per band: load the float64 carries, then one top-down sweep.  In-band arithmetic
// in A (float32 when the field is stored as float32), carries rounded to A once.
#ifndef DET_SAT3_PIPE
#define DET_SAT3_PIPE 0  // 1: 53.6k vs 54.7k (spills at the 64-register cap)
#endif
#ifndef DET_SAT3_F2
#define DET_SAT3_F2 1
#endif
#ifndef DET_SAT3_ABS
#define DET_SAT3_ABS 1  // float64 field: anchor case splits as |e|, |d| terms (no compares/selects)
#endif
#ifndef DET_SAT3_MINB
#define DET_SAT3_MINB 4  // 64 registers, no spills: 512 band CTAs fit one wave (3 and 5 measured slower)
#endif
#ifndef DET_SAT3_MINB64
#define DET_SAT3_MINB64 2  // float64 in-band arithmetic: up to 128 registers (64 spill ~300 bytes)
#endif
template <int CPT, int NT, int SRC, typename UT, int OUT, typename A, bool LUTS>
__global__ void __launch_bounds__(NT, (NT <= 256 ? (sizeof(A) == 8 ? DET_SAT3_MINB64 : DET_SAT3_MINB) : 1))
    k_sat3(Topo T, Bufs D, SatSrc S, int gate) {
    extern __shared__ unsigned char s_raw3[];
    constexpr int NW = NT / 32;
    __shared__ A s_w[3][32];
    __shared__ A s_xa[3][32], s_xu1[3][32], s_xu2[3][32], s_xr[3][32];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, M = 2 * n - 1, R = T.R;
    const int x0 = t * CPT;
    const bool active = x0 < n;  // n is a multiple of CPT: a thread's columns are all in or all out
    const size_t bb = (size_t)b * D.nb + band;
    const int WN = n + H;
    // DLtot(w) and Tu(w) interleaved, w in [jt-1, jb+n-1] -> [w-(jt-1)]: one 2-wide load per w
    using A2 = typename std::conditional<sizeof(A) == 4, float2, double2>::type;
    A2* win_dt = reinterpret_cast<A2*>(s_raw3);
    A* win_tv = reinterpret_cast<A*>(win_dt + WN);  // Tv(v), v in [-jb, n-1-jt] -> [v+jb]
    A* s_rc = win_tv + WN;                          // per band row: ravg, rowfull(j+1), right boundary
    A* s_lut = s_rc + 3 * H + (H & 1);
    const double* rowfull = D.rowfull + (size_t)b * (n + 1);
    const double* adT = D.adT + (size_t)b * M;
    const double* dgT = D.dgT + (size_t)b * M;
    const double* csT = D.csT + (size_t)b * n;

    // ---- carries (k_sat2), row constants, LUT ----
#pragma unroll 4
    for (int q = t; q < WN; q += blockDim.x) {
        win_dt[q].x = (jt == 0 && q == 0) ? (A)0 : (A)D.adSc[bb * WN + q];  // DLtot(-1) = 0
        const int wq = jt - 1 + q;
        win_dt[q].y = (wq >= 0 && wq < M) ? (A)adT[wq] : (A)0;  // Tu(w), defined up to jb+n-2
        const int iv = q - jb + n - 1;  // Tv index of v = q - jb
        win_tv[q] = (iv >= 0 && iv < M) ? (A)dgT[iv] : (A)0;
    }
    const double rf_top = rowfull[jt];
    for (int q = t; q < H; q += blockDim.x) {
        const double r0 = rowfull[jt + q], r1 = rowfull[jt + q + 1];
        s_rc[q] = (A)(0.5 * (r0 + r1));
        s_rc[H + q] = (A)r1;
        s_rc[2 * H + q] = (A)(r0 - rf_top);
    }
    // float ring path: background-first shared LUT, labels index it directly (band_lut BIAS)
    // labels through the shared-memory TMA ring (float path; float64 path up to 4096 columns --
    // at 8192 its carry windows leave no room); register prefetch otherwise
    constexpr bool RING = SRC == SRC_LABELS && OUT == OUT_U && (sizeof(A) == 4 || CPT * NT <= 4096);
    constexpr bool LB = LUTS && RING;
    const A* lut = band_lut<A, LUTS, LB>(D, R, b, s_lut);
    // cc[k]: column-total average cavg(x) = (colfull(x) + colfull(x+1))/2 for the field,
    // colfull(x+1) for the channel dump
    // PF (float32 field): al[k] carries the column-pair sum alpha(j-1, x-1) + alpha(j-1, x) instead
    // of alpha itself -- each thread advances it from its own row prefixes, so the straight
    // channel needs no neighbour exchange and a = (pair(j-1) + pair(j)) / 4
    constexpr bool PF = OUT == OUT_U && sizeof(A) == 4;
    A ul[CPT], al[CPT], cc[CPT], ur[CPT];
    A al_left = (PF && x0 > 0 && active) ? (A)D.csX[bb * n + x0 - 1] : (A)0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        const bool in = x < n;
        al[k] = in ? (A)D.csX[bb * n + x] : (A)0;
        if (PF) {
            const A t = al[k];
            al[k] = al_left + t;
            al_left = t;
        }
        ul[k] = in ? (A)D.dgXc[bb * n + x] : (A)0;
        const double cfi = in ? csT[x] : 0.0, cfe = (in && x > 0) ? csT[x - 1] : 0.0;
        cc[k] = (A)(OUT == OUT_CH8 ? cfi : 0.5 * (cfe + cfi));
        ur[k] = (A)0;
    }
    if (lane == 31) {  // boundary values of "row jt-1" = carries
        if (!PF) s_xa[2][w] = al[CPT - 1];
        s_xu1[2][w] = ul[CPT - 1];
        s_xu2[2][w] = ul[CPT - 2];
    }
    if (lane == 0) s_xr[2][w] = (A)0;
    const A Cr = (A)rowfull[n];
    const double inv_nd = 1.0 / (double)n;  // exact: n is a power of two
    const A inv_n = (A)inv_nd, half_n = (A)(0.5 * inv_nd);
    const A inv2m = (A)(S.outscale != 0.0 ? S.outscale : 0.5 * inv_nd * inv_nd);
    const A xc0 = (A)(((double)x0 + 0.5) * inv_nd);  // pixel-centre x of column x0 (displacement.py:59)
    UT* uf = reinterpret_cast<UT*>(D.uf) + (size_t)b * D.nn * 2;
    __shared__ uint64_t s_bar[4];
    LabelRing<CPT, lab_kp(CPT * NT)> ring;
    if (RING) {
        ring.q = align16(s_lut + (LUTS ? lut_smem_len(R) : 0));
        ring.bar = s_bar;
        ring.lab = D.labels + (size_t)b * D.nn;
        ring.stride = NT * CPT;
        ring.n = n;
        ring.x0 = x0;
        ring.jt = jt;
        ring.j_last = jb;
        ring.active = active;
        ring.init();
    }
    __syncthreads();  // windows, row constants, LUT and the ring's mbarriers published
    if (RING) ring.prologue();
    A rho_n[CPT];
    if (!RING) load_rho<CPT, SRC, A, LUTS>(D, S, lut, R, b, jt, x0, rho_n);
    // DET_SAT3_PIPE: row j+1's label wait and LUT reads are issued at the top of row j (as in k_sat1)
    if (RING && DET_SAT3_PIPE) ring.template take<A, LB>(jt, lut, R, rho_n);

    int slot = 0, ps = 2;  // rotating boundary slots: (j - jt) % 3, (j - jt + 2) % 3
    for (int j = jt; j <= jb; ++j) {
        A rho[CPT];
        if (RING && DET_SAT3_PIPE) {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
            if (j < jb) ring.template take<A, LB>(j + 1, lut, R, rho_n);  // refills row j's slot: every take(j) preceded barrier j-1
        } else if (RING) {
            ring.template take<A, LB>(j, lut, R, rho);
        } else {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
            if (j < jb) load_rho<CPT, SRC, A, LUTS>(D, S, lut, R, b, j + 1, x0, rho_n);  // prefetch the next row
        }
        A loc[CPT];
        A run = (A)0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) { run += rho[k]; loc[k] = run; }
        // A(j, x0-1): in-warp scan of the thread sums, then a scan of the warp totals
        const A tsum = run;
        const A winc = warp_incl_scan_t<A>(tsum);
        if (lane == 31) s_w[slot][w] = winc;
        __syncthreads();
        A wt = lane < NW ? s_w[slot][lane] : (A)0;
        // scan of the NW warp totals: log2(NW) steps, not a full 32-lane scan
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) {
            const A tt = __shfl_up_sync(FULL, wt, o);
            if (lane >= o) wt += tt;
        }
        const A woff = __shfl_sync(FULL, wt, (w + 31) & 31);
        const A excl = (w == 0 ? (A)0 : woff) + winc - tsum;
        A ap_m1 = PF ? (A)0 : __shfl_up_sync(FULL, al[CPT - 1], 1);
        A ul_m1 = __shfl_up_sync(FULL, ul[CPT - 1], 1);
        A ul_m2 = __shfl_up_sync(FULL, ul[CPT - 2], 1);
        A ur_p = __shfl_down_sync(FULL, ur[0], 1);
        if (lane == 0) {
            if (w == 0) { ap_m1 = (A)0; ul_m1 = (A)0; ul_m2 = (A)0; }
            else { if (!PF) ap_m1 = s_xa[ps][w - 1]; ul_m1 = s_xu1[ps][w - 1]; ul_m2 = s_xu2[ps][w - 1]; }
        }
        if (lane == 31) ur_p = (w == NW - 1) ? s_rc[2 * H + (j - jt)] : s_xr[ps][w + 1];
        A Av[CPT], an[CPT], uln[CPT], urn[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) Av[k] = excl + loc[k];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            // PF: the new column-pair sum (A(j, x-1) + A(j, x) added; A(j, x0-1) = excl)
            an[k] = PF ? al[k] + ((k == 0 ? excl : Av[k - 1]) + Av[k]) : al[k] + Av[k];
            uln[k] = Av[k] + (k == 0 ? ul_m1 : ul[k - 1]);
            urn[k] = Av[k] + (k == CPT - 1 ? ur_p : ur[k + 1]);
        }
        if (active) {
            const A ravg = s_rc[j - jt], rf1 = s_rc[H + (j - jt)];
            const A yc = (A)j * inv_n + half_n;  // (j + 0.5) / n, exact in A
            // PF row constants: y - 1, (1 - 2y) / 4, ravg - C
            const A ycm1 = yc - (A)1, c1y = (A)0.25 - (A)0.5 * yc, rmc = ravg - Cr;
            const A hravg = (A)0.5 * ravg, hC = (A)0.5 * Cr;  // float64 branch-free form
            const int wi0 = j + x0 - (jt - 1);
            A dlw[CPT + 1];  // DLtot(j + x - 1 + q), sliding window over this thread's columns
            A tuw[CPT];      // Tu(j + x - 1 + q)
#pragma unroll
            for (int q = 0; q <= CPT; ++q) {
                const A2 v = win_dt[wi0 - 1 + q];
                dlw[q] = v.x;
                if (q < CPT) tuw[q] = v.y;
            }
            A ux[CPT], uy[CPT];
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int x = x0 + k;
                const A apm1 = k == 0 ? ap_m1 : al[k - 1];
                const A anm1 = k == 0 ? (ap_m1 + excl) : an[k - 1];
                const A ulnm1 = k == 0 ? (excl + ul_m2) : uln[k - 1];
                const A ulpm1 = k == 0 ? ul_m1 : ul[k - 1];
                const A ulpm2 = k == 0 ? ul_m2 : (k == 1 ? ul_m1 : ul[k - 2]);
                const A urp1 = k == CPT - 1 ? ur_p : ur[k + 1];
                const A Dw = dlw[k + 1], Dwm1 = dlw[k];
                const A Tu = tuw[k];
                const A Tv = win_tv[x - j + jb];
                const A R_UV = ulpm1 + (Dw - urp1);
                A R_UVm1 = ulnm1 + (Dw - urn[k]);
                A R_Um1Vm1 = ulpm2 + (Dwm1 - ur[k]);
                if (k == 0 && x0 == 0) { R_UVm1 = (A)0; R_Um1Vm1 = (A)0; }
                const A bt = R_UVm1;
                const A at = Tu - R_Um1Vm1 + rho[k];
                const A gt = Tv - R_UV;
                if (OUT == OUT_CH8) {
                    const A dt = Cr - at - bt - gt;
                    double* ch = S.ch8 + (size_t)b * 8 * D.nn + (size_t)j * n + x;
                    const size_t nn = D.nn;
                    ch[0] = an[k];
                    ch[nn] = cc[k] - an[k];
                    ch[2 * nn] = Cr - cc[k] - rf1 + an[k];
                    ch[3 * nn] = rf1 - an[k];
                    ch[4 * nn] = at;
                    ch[5 * nn] = bt;
                    ch[6 * nn] = gt;
                    ch[7 * nn] = dt;
                } else if constexpr (PF) {
                    // the same anchor combination with the case splits of displacement.py:62,67 as
                    // min/max: with e = x + y - 1 and d = x - y,
                    //   q2x = q4y = 1 + min(e, 0),  q2y = q4x = max(e, 0),  q3 = (max(d, 0), max(-d, 0))
                    const A a4 = al[k] + an[k];  // 4a
                    const A cavg = cc[k];
                    const A xc = xc0 + (A)k * inv_n;
                    const A e = xc + ycm1, d = xc - yc;
                    const A mn = fminf(e, (A)0), mx = fmaxf(e, (A)0);
                    const A dp = fmaxf(d, (A)0), dn = fmaxf(-d, (A)0);
                    const A nK = -(cavg + rmc);
                    const A t = at + gt;
#if DET_SAT3_F2
                    // (ux, uy) as one packed pair: FFMA2 / FADD2 / FMUL2 (sm_100 f32x2)
                    float2 v = __ffma2_rn(make_float2(a4, a4), make_float2(c1y, fmaf(xc, -0.5f, 0.25f)),
                                          make_float2(cavg, ravg));
                    v = __ffma2_rn(make_float2(cavg, cavg), make_float2(mn, mx), v);
                    v = __ffma2_rn(make_float2(ravg, ravg), make_float2(mx, mn), v);
                    v = __ffma2_rn(make_float2(nK, nK), make_float2(dp, dn), v);
                    v = __ffma2_rn(make_float2(xc, yc), make_float2(t, Cr - t), v);
                    v = __fmul2_rn(__fadd2_rn(v, make_float2(bt, at)), make_float2(inv2m, inv2m));
                    ux[k] = v.x;
                    uy[k] = v.y;
#else
                    A vx = fmaf(a4, c1y, cavg);
                    vx = fmaf(cavg, mn, vx);
                    vx = fmaf(ravg, mx, vx);
                    vx = fmaf(nK, dp, vx);
                    vx = fmaf(xc, t, vx);
                    ux[k] = (vx + bt) * inv2m;
                    A vy = fmaf(a4, fmaf(xc, (A)-0.5, (A)0.25), ravg);
                    vy = fmaf(cavg, mx, vy);
                    vy = fmaf(ravg, mn, vy);
                    vy = fmaf(nK, dn, vy);
                    vy = fmaf(yc, Cr - t, vy);
                    uy[k] = (vy + at) * inv2m;
#endif
                } else if constexpr (OUT == OUT_U && sizeof(A) == 8 && DET_SAT3_ABS) {
                    // float64 field, branch-free: with e = x + y - 1 and d = x - y the case splits
                    // of displacement.py:62,67 are q2x = q4y = 1 + (e - |e|)/2, q2y = q4x = (e + |e|)/2,
                    // q3 = ((d + |d|)/2, (|d| - d)/2), so the combination below needs no compares or
                    // selects: ux*2m = a(1-2y) + cavg + hs e + hd |e| - hK (d + |d|) + x t + bt,
                    // uy*2m = a(1-2x) + ravg + hs e - hd |e| + hK (d - |d|) + at + y (C - t) with
                    // hs = (cavg + ravg)/2, hd = (ravg - cavg)/2, hK = (cavg + ravg - C)/2
                    const A a4 = apm1 + al[k] + anm1 + an[k];  // 4a
                    const A cavg = cc[k];
                    const A xc = xc0 + (A)k * inv_n;
                    const A e = xc + ycm1, d = xc - yc;
                    const A ae = fabs(e), ad = fabs(d);
                    const A hs = fma((A)0.5, cavg, hravg), hd = fma((A)-0.5, cavg, hravg);
                    const A hK = hs - hC;
                    const A t = at + gt;
                    A vx = fma(a4, c1y, cavg);
                    vx = fma(hs, e, vx);
                    vx = fma(hd, ae, vx);
                    vx = fma(-hK, d + ad, vx);
                    vx = fma(xc, t, vx);
                    ux[k] = (vx + bt) * inv2m;
                    A vy = fma(a4, fma(xc, (A)-0.5, (A)0.25), ravg);
                    vy = fma(hs, e, vy);
                    vy = fma(-hd, ae, vy);
                    vy = fma(hK, d - ad, vy);
                    vy = fma(yc, Cr - t, vy);
                    uy[k] = (vy + at) * inv2m;
                } else {
                    // anchor combination (displacement.py:128-130) with b = cavg-a, d = ravg-a,
                    // g = C-cavg-ravg+a, delta_t = C-at-bt-gt; since q1+q3 = (1+x-y, 1-x+y) and
                    // q2+q4 = (x+y, x+y) in every case, a's coefficient is (1-2y, 1-2x).
                    const A a = (A)0.25 * (apm1 + al[k] + anm1 + an[k]);
                    const A cavg = cc[k];
                    const A K = cavg + ravg - Cr;
                    const A xc = xc0 + (A)k * inv_n, s2 = xc + yc;
                    const bool below = yc < xc, near = s2 < (A)1;  // displacement.py:62,67
                    const A q3x = below ? xc - yc : (A)0, q3y = below ? (A)0 : yc - xc;
                    const A q2x = near ? s2 : (A)1, q2y = near ? (A)0 : s2 - (A)1;
                    const A q4x = near ? (A)0 : s2 - (A)1, q4y = near ? s2 : (A)1;
                    ux[k] = (a * ((A)1 - (A)2 * yc) + cavg * q2x + ravg * q4x - K * q3x + xc * (at + gt) + bt) * inv2m;
                    uy[k] = (a * ((A)1 - (A)2 * xc) + cavg * q2y + ravg * q4y - K * q3y + at + yc * (Cr - at - gt)) * inv2m;
                }
            }
            if (OUT != OUT_CH8) {
                UT* o = uf + ((size_t)j * n + x0) * 2;
                if (sizeof(UT) == 8 && CPT % 2 == 0) {  // two float64 pixels per 32-byte store (whole sectors)
#pragma unroll
                    for (int k = 0; k < CPT; k += 2)
                        st_global_v4f64(o + 2 * k, (double)ux[k], (double)uy[k], (double)ux[k + 1], (double)uy[k + 1]);
                } else if (sizeof(UT) == 4 && CPT % 4 == 0) {  // four float32 pixels per 32-byte store
#pragma unroll
                    for (int k = 0; k < CPT; k += 4)
                        st_global_v8f32(o + 2 * k, (float)ux[k], (float)uy[k], (float)ux[k + 1], (float)uy[k + 1],
                                        (float)ux[k + 2], (float)uy[k + 2], (float)ux[k + 3], (float)uy[k + 3]);
                } else if (sizeof(UT) == 4 && CPT % 2 == 0) {  // two pixels per 16-byte store
#pragma unroll
                    for (int k = 0; k < CPT; k += 2)
                        *reinterpret_cast<float4*>(o + 2 * k) =
                            make_float4((float)ux[k], (float)uy[k], (float)ux[k + 1], (float)uy[k + 1]);
                } else {
#pragma unroll
                    for (int k = 0; k < CPT; ++k) {
                        o[2 * k] = (UT)ux[k];
                        o[2 * k + 1] = (UT)uy[k];
                    }
                }
            }
        }
        if (lane == 31) {
            if (!PF) s_xa[slot][w] = an[CPT - 1];
            s_xu1[slot][w] = uln[CPT - 1];
            s_xu2[slot][w] = uln[CPT - 2];
        }
        if (lane == 0) s_xr[slot][w] = urn[0];
#pragma unroll
        for (int k = 0; k < CPT; ++k) { al[k] = an[k]; ul[k] = uln[k]; ur[k] = urn[k]; }
        ps = slot;
        slot = slot == 2 ? 0 : slot + 1;
    }
}


// ---------------------------------------------------------------------------------
// k_sat3w: k_sat3 for the float64 field with independent warps and no CTA barrier in the sweep.
// A CTA covers a band and up to 32*CPT*NT/32 columns (cb = its first column); each warp owns a
// W = 32*CPT column slice and streams it through its own TMA ring.  What crosses a slice edge in
// row j = jt + r is formed from k_sat1w's slice tables (off, E1, exD, exA; see k_sat1w TAB) instead
// of being exchanged between warps:
//   A(j, c0-1)       = off(r, w)
//   alpha(j-1, c0-1) = csX(c0-1) + sum_{r'<r} off(r', w)
//   UL(j-1, c0-1)    = dgXc(c0-1-r) + sum_{r'<r} off(r', w-1) + E1(r-1, w-1)
//   UL(j-1, c0-2)    = dgXc(c0-2-r) + sum_{r'<r} off(r', w-1) + E1(r-1, w-1) - exD(r-1, w-1)
//   URin(j-1, c0+W)  = sum_{r'<r} (off(r', w+1) + exA(r', w+1))
// (H <= W - 1: every diagonal / anti-diagonal through a band crosses at most one slice edge, so its
// in-band sum left / right of the edge is the neighbour slice's in-slice partial.)  The per-pixel
// arithmetic is k_sat3's float64 anchor combination (displacement.py:102-131 in residual form).
template <int CPT, int NT, bool LUTS>
__global__ void __launch_bounds__(NT, (NT <= 256 ? DET_SAT3_MINB64 : 1)) k_sat3w(Topo T, Bufs D, int gate) {
    using A = double;
    extern __shared__ unsigned char s_raw3w[];
    constexpr int NWC = NT / 32, W = 32 * CPT, KP = lab_kp(W * NWC) > 4 ? 4 : lab_kp(W * NWC);
    __shared__ uint64_t s_bar[NWC * KP];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, wl = t >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, M = 2 * n - 1, R = T.R;
    const int NW = n / W;                   // slices per band row
    const int cb = blockIdx.z * NWC * W;    // this CTA's first column
    const int w = blockIdx.z * NWC + wl;    // slice index in the band row
    const int c0 = w * W, x0 = c0 + lane * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    const int WN = NWC * W + H;
    // The windows are stored phase-split, element e at [e % 4][e / 4] (P entries per phase): lane l
    // reads elements e0 + 4l + q, so every load of a warp touches consecutive words of one phase
    // (bank-conflict-free) instead of a 4-element stride (16-way conflicts on 16-byte loads).
    const int P = (WN + 3) / 4 + 1;
    using A2 = double2;
    A2* win_dt = reinterpret_cast<A2*>(s_raw3w);  // DLtot(w), Tu(w) for w in [cb+jt-1, cb+jb+NWC*W-1]
    A* win_tv = reinterpret_cast<A*>(win_dt + 4 * P);  // Tv(v), v in [cb-jb, cb+NWC*W-1-jt]
    A* s_rc = win_tv + 4 * P;                       // per band row: ravg, rowfull(j+1), right boundary
    A* s_tab = s_rc + 3 * H + (H & 1);              // [4][NWC + 2][H]: slices cb/W - 1 .. cb/W + NWC
    A* s_cw = s_tab + 4 * (NWC + 2) * H;            // [NWC][H + 1]: dgXc(c0 - 1 - m)
    A* s_lut = s_cw + NWC * (H + 1) + ((NWC * (H + 1)) & 1);
    const double* rowfull = D.rowfull + (size_t)b * (n + 1);
    const double* adT = D.adT + (size_t)b * M;
    const double* dgT = D.dgT + (size_t)b * M;
    const double* csT = D.csT + (size_t)b * n;
    const double* tabg = D.tab + bb * 4 * NW * H;

    // ---- carries (k_sat2p), slice tables, row constants, LUT ----
    for (int q = t; q < WN; q += NT) {
        const int wq = cb + jt - 1 + q;
        const int ps = (q & 3) * P + (q >> 2);
        win_dt[ps].x = (wq < 0) ? 0.0 : D.adSc[bb * (n + H) + (q + cb)];  // DLtot(-1) = 0
        win_dt[ps].y = (wq >= 0 && wq < M) ? adT[wq] : 0.0;
        const int iv = q + cb - jb + n - 1;  // Tv index of v = q + cb - jb
        win_tv[ps] = (iv >= 0 && iv < M) ? dgT[iv] : 0.0;
    }
    for (int i = t; i < 4 * (NWC + 2) * H; i += NT) {
        const int f = i / ((NWC + 2) * H), rem = i - f * (NWC + 2) * H, sl = rem / H, r = rem - sl * H;
        const int ws = cb / W - 1 + sl;
        s_tab[i] = (ws >= 0 && ws < NW) ? tabg[(f * NW + ws) * H + r] : 0.0;
    }
    for (int i = t; i < NWC * (H + 1); i += NT) {
        const int sl = i / (H + 1), m = i - sl * (H + 1);
        const int x = cb + sl * W - 1 - m;
        s_cw[i] = x >= 0 ? D.dgXc[bb * n + x] : 0.0;
    }
    const double rf_top = rowfull[jt];
    for (int q = t; q < H; q += NT) {
        const double r0 = rowfull[jt + q], r1 = rowfull[jt + q + 1];
        s_rc[q] = 0.5 * (r0 + r1);
        s_rc[H + q] = r1;
        s_rc[2 * H + q] = r0 - rf_top;
    }
    const A* lut = band_lut<A, LUTS, LUTS>(D, R, b, s_lut);
    A ul[CPT], al[CPT], cc[CPT], ur[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        al[k] = D.csX[bb * n + x];
        ul[k] = D.dgXc[bb * n + x];
        const double cfi = csT[x], cfe = x > 0 ? csT[x - 1] : 0.0;
        cc[k] = 0.5 * (cfe + cfi);
        ur[k] = 0.0;
    }
    A aL = c0 > 0 ? D.csX[bb * n + c0 - 1] : 0.0;  // alpha(j-1, c0-1), advanced per row
    A sL = 0.0, sR = 0.0;                            // running sums of the neighbour tables
    const A Cr = rowfull[n];
    const double inv_nd = 1.0 / (double)n;  // exact: n is a power of two
    const A inv_n = inv_nd, half_n = 0.5 * inv_nd;
    const A inv2m = 0.5 * inv_nd * inv_nd;
    const A xc0 = ((double)x0 + 0.5) * inv_nd;  // pixel-centre x of column x0 (displacement.py:59)
    double* uf = reinterpret_cast<double*>(D.uf) + (size_t)b * D.nn * 2;
    WarpRing<CPT, KP> ring;
    ring.q = align16(s_lut + (LUTS ? lut_smem_len(R) : 0)) + wl * KP * W;
    ring.bar = s_bar + wl * KP;
    ring.lab = D.labels + (size_t)b * D.nn + c0;
    ring.n = n;
    ring.jt = jt;
    ring.j_last = jb;
    ring.bytes = (unsigned)(W * 4);
    ring.init(lane);
    ring.prologue(lane);
    __syncthreads();  // windows, tables, row constants and LUT published (the only CTA barrier)
    const A* tO = s_tab + (wl + 1) * H;                // own slice: off
    const A* tOL = s_tab + wl * H;                     // left slice: off, E1 (+ (NWC+2)H), exD (+ 2(NWC+2)H)
    const A* tOR = s_tab + (wl + 2) * H;               // right slice: off, exA (+ 3(NWC+2)H)
    constexpr int dummy = 0;
    (void)dummy;
    const int FS = (NWC + 2) * H;
    const A* cw = s_cw + wl * (H + 1);
    const bool first = w == 0, last = w == NW - 1;

    for (int j = jt; j <= jb; ++j) {
        const int r = j - jt;
        A rho[CPT];
        ring.template take<A, LUTS>(j, lane, true, lut, R, rho);
        // edge values of row j-1 from the tables (running sums advanced by row r-1)
        A e1 = 0.0, exd = 0.0;
        if (r > 0) {
            aL += tO[r - 1];
            sL += tOL[r - 1];
            sR += tOR[r - 1];
            sR += tOR[3 * FS + r - 1];
            e1 = tOL[FS + r - 1];
            exd = tOL[2 * FS + r - 1];
        }
        const A base = first ? 0.0 : tO[r];  // A(j, c0-1)
        A loc[CPT];
        A run = 0.0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) { run += rho[k]; loc[k] = run; }
        const A tsum = run;
        const A winc = warp_incl_scan_t<A>(tsum);
        const A excl = base + (winc - tsum);
        A ap_m1 = __shfl_up_sync(FULL, al[CPT - 1], 1);
        A ul_m1 = __shfl_up_sync(FULL, ul[CPT - 1], 1);
        A ul_m2 = __shfl_up_sync(FULL, ul[CPT - 2], 1);
        A ur_p = __shfl_down_sync(FULL, ur[0], 1);
        if (lane == 0) {
            if (first) { ap_m1 = 0.0; ul_m1 = 0.0; ul_m2 = 0.0; }
            else {
                const A le = sL + e1;
                ap_m1 = aL;
                ul_m1 = cw[r] + le;
                ul_m2 = cw[r + 1] + (le - exd);
            }
        }
        if (lane == 31) ur_p = last ? s_rc[2 * H + r] : sR;
        A Av[CPT], an[CPT], uln[CPT], urn[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) Av[k] = excl + loc[k];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            an[k] = al[k] + Av[k];
            uln[k] = Av[k] + (k == 0 ? ul_m1 : ul[k - 1]);
            urn[k] = Av[k] + (k == CPT - 1 ? ur_p : ur[k + 1]);
        }
        {
            const A ravg = s_rc[r];
            const A yc = (A)j * inv_n + half_n;  // (j + 0.5) / n, exact
            const A ycm1 = yc - 1.0, c1y = 0.25 - 0.5 * yc;
            const A hravg = 0.5 * ravg, hC = 0.5 * Cr;
            const int e0 = j - jt + c0 - cb;  // window element of lane 0's dlw[0]: e0 + CPT*lane + q
            const int f0 = c0 - cb - j + jb;  // win_tv element of lane 0's column c0: f0 + CPT*lane + k
            A dlw[CPT + 1];
            A tuw[CPT], tvw[CPT];
#pragma unroll
            for (int q = 0; q <= CPT; ++q) {
                const int e = e0 + q;
                const A2 v = win_dt[(e & 3) * P + (e >> 2) + lane];
                dlw[q] = v.x;
                if (q < CPT) tuw[q] = v.y;
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int e = f0 + k;
                tvw[k] = win_tv[(e & 3) * P + (e >> 2) + lane];
            }
            A ux[CPT], uy[CPT];
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int x = x0 + k;
                const A apm1 = k == 0 ? ap_m1 : al[k - 1];
                const A anm1 = k == 0 ? (ap_m1 + excl) : an[k - 1];
                const A ulnm1 = k == 0 ? (excl + ul_m2) : uln[k - 1];
                const A ulpm1 = k == 0 ? ul_m1 : ul[k - 1];
                const A ulpm2 = k == 0 ? ul_m2 : (k == 1 ? ul_m1 : ul[k - 2]);
                const A urp1 = k == CPT - 1 ? ur_p : ur[k + 1];
                const A Dw = dlw[k + 1], Dwm1 = dlw[k];
                const A Tu = tuw[k];
                const A Tv = tvw[k];
                const A R_UV = ulpm1 + (Dw - urp1);
                A R_UVm1 = ulnm1 + (Dw - urn[k]);
                A R_Um1Vm1 = ulpm2 + (Dwm1 - ur[k]);
                if (k == 0 && x0 == 0) { R_UVm1 = 0.0; R_Um1Vm1 = 0.0; }
                const A bt = R_UVm1;
                const A at = Tu - R_Um1Vm1 + rho[k];
                const A gt = Tv - R_UV;
                // branch-free anchor combination (see k_sat3, DET_SAT3_ABS)
                const A a4 = apm1 + al[k] + anm1 + an[k];  // 4a
                const A cavg = cc[k];
                const A xc = xc0 + (A)k * inv_n;
                const A e = xc + ycm1, d = xc - yc;
                const A ae = fabs(e), ad = fabs(d);
                const A hs = fma(0.5, cavg, hravg), hd = fma(-0.5, cavg, hravg);
                const A hK = hs - hC;
                const A tt = at + gt;
                A vx = fma(a4, c1y, cavg);
                vx = fma(hs, e, vx);
                vx = fma(hd, ae, vx);
                vx = fma(-hK, d + ad, vx);
                vx = fma(xc, tt, vx);
                ux[k] = (vx + bt) * inv2m;
                A vy = fma(a4, fma(xc, -0.5, 0.25), ravg);
                vy = fma(hs, e, vy);
                vy = fma(-hd, ae, vy);
                vy = fma(hK, d - ad, vy);
                vy = fma(yc, Cr - tt, vy);
                uy[k] = (vy + at) * inv2m;
            }
            double* o = uf + ((size_t)j * n + x0) * 2;
#pragma unroll
            for (int k = 0; k < CPT; k += 2) st_global_v4f64(o + 2 * k, ux[k], uy[k], ux[k + 1], uy[k + 1]);
        }
#pragma unroll
        for (int k = 0; k < CPT; ++k) { al[k] = an[k]; ul[k] = uln[k]; ur[k] = urn[k]; }
    }
}

// ---------------------------------------------------------------------------------
// k_sat3x: k_sat3w with everything that does not depend on the pixel taken out of the row loop.
//  * The values crossing a slice edge (k_sat3w's running sums over k_sat1w's slice tables) are
//    prefixed once per band by the warp itself (a warp scan over the band rows) into a 6-double
//    record per row -- A(j, c0-1), alpha(j-1, c0-1), UL(j-1, c0-1), UL(j-1, c0-2), URin(j-1, c0+W)
//    and the row-total average -- which the row reads as three broadcast 16-byte loads.
//  * The row loop is unrolled four times, so the phase of the phase-split carry windows, the ring
//    slot and the record offset are compile-time: every shared load of a row is [pointer + immediate],
//    the pointers advance once per four rows, and the carries rotate by register renaming.
// The per-pixel arithmetic is k_sat3w's, in the same operation order (the edge prefixes are summed
// in warp-scan order instead of row order).  CPT = 4 only (KP = 4 ring slots = the unroll).
#ifndef DET_SAT3X_PIPE
#define DET_SAT3X_PIPE 0  // 2: the next row's row-prefix scan issued ahead of this row's field arithmetic, densities re-read (54.3k vs 55.4k it/s); 1: the next row's labels, LUT reads and row-prefix scan issued ahead of this row's field arithmetic (spills at 128 registers: 49.6k vs 51.6k it/s)
#endif
// FA (band-fused advect, fa_par = iteration parity >= 0): after the sweep the CTA advects the unique
// vertices whose bilinear tap lies inside this band (advect_band_vertices, det_raster.cuh) while the
// band's field rows are still on chip; the CTA must span the whole band row (gridDim.z == 1).
template <int NT, bool LUTS, bool FA = false>
__global__ void __launch_bounds__(NT, (NT <= 256 ? DET_SAT3_MINB64 : 1)) k_sat3x(Topo T, Bufs D, int gate, int fa_par = -1,
                                                                                 const int* __restrict__ uq_off = nullptr) {
    using A = double;
    using A2 = double2;
    constexpr int CPT = 4, NWC = NT / 32, W = 32 * CPT, KP = 4;
    constexpr int P = sat3x_phase_len(NWC);  // entries per window phase (compile-time: H < W)
    extern __shared__ __align__(16) unsigned char s_raw3x[];
    __shared__ uint64_t s_bar[NWC * KP];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, wl = t >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, M = 2 * n - 1, R = T.R;
    const int NW = n / W;                   // slices per band row
    const int cb = blockIdx.z * NWC * W;    // this CTA's first column
    const int w = blockIdx.z * NWC + wl;    // slice index in the band row
    const int c0 = w * W, x0 = c0 + lane * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    const int WN = NWC * W + H;
    const int pad = (3 - (H - 1)) & 3;      // win_tv storage shift: row r reads phase (3 - r + k) & 3
    const int Hq = (H - 1 + pad) >> 2;
    A2* win_dt = reinterpret_cast<A2*>(s_raw3x);       // [4][P]: DLtot(w), Tu(w), w from cb+jt-1, element e at [e&3][e>>2]
    A* win_tv = reinterpret_cast<A*>(win_dt + 4 * P);  // [4][P]: Tv(v), v from cb-jb, element e+pad at [..&3][..>>2]
    A* s_rec = win_tv + 4 * P;                         // [NWC][H][6] edge records
    A* s_lut = s_rec + (size_t)NWC * H * 6;
    const double* rowfull = D.rowfull + (size_t)b * (n + 1);
    const double* adT = D.adT + (size_t)b * M;
    const double* dgT = D.dgT + (size_t)b * M;
    const double* csT = D.csT + (size_t)b * n;
    const double* tabg = D.tab + bb * 4 * NW * H;

    // ---- carries (k_sat2p) into the phase-split windows, LUT ----
    for (int q = t; q < WN; q += NT) {
        const int wq = cb + jt - 1 + q;
        A2 v;
        v.x = (wq < 0) ? 0.0 : D.adSc[bb * (n + H) + (q + cb)];  // DLtot(-1) = 0
        v.y = (wq >= 0 && wq < M) ? adT[wq] : 0.0;
        win_dt[(q & 3) * P + (q >> 2)] = v;
        const int iv = q + cb - jb + n - 1;  // Tv index of v = q + cb - jb
        const int qp = q + pad;
        win_tv[(qp & 3) * P + (qp >> 2)] = (iv >= 0 && iv < M) ? dgT[iv] : 0.0;
    }
    const A* lut = band_lut<A, LUTS, LUTS>(D, R, b, s_lut);
    // ---- this warp's edge records: exclusive prefixes over the band rows of the slice tables ----
    {
        const bool first = w == 0, last = w == NW - 1;
        const double rf_top = rowfull[jt];
        A cA = c0 > 0 ? D.csX[bb * n + c0 - 1] : 0.0;  // alpha(jt-1, c0-1)
        A cL = 0.0, cR = 0.0;
        A* rec = s_rec + (size_t)wl * H * 6;
        for (int r0 = 0; r0 < H; r0 += 32) {
            const int r = r0 + lane;
            const bool in = r < H;
            const A offw = (in && !first) ? tabg[(0 * NW + w) * H + r] : 0.0;
            const A offl = (in && !first) ? tabg[(0 * NW + w - 1) * H + r] : 0.0;
            const A offr = (in && !last) ? tabg[(0 * NW + w + 1) * H + r] + tabg[(3 * NW + w + 1) * H + r] : 0.0;
            const A sA = warp_incl_scan_t<A>(offw), sL = warp_incl_scan_t<A>(offl), sR = warp_incl_scan_t<A>(offr);
            if (in) {
                const A e1 = (!first && r > 0) ? tabg[(1 * NW + w - 1) * H + r - 1] : 0.0;
                const A exd = (!first && r > 0) ? tabg[(2 * NW + w - 1) * H + r - 1] : 0.0;
                const int xa = c0 - 1 - r;
                const A cw0 = xa >= 0 ? D.dgXc[bb * n + xa] : 0.0;
                const A cw1 = xa >= 1 ? D.dgXc[bb * n + xa - 1] : 0.0;
                const A le = (cL + (sL - offl)) + e1;
                const double rf0 = rowfull[jt + r], rf1 = rowfull[jt + r + 1];
                A* o = rec + r * 6;
                o[0] = offw;                                         // A(j, c0-1)
                o[1] = first ? 0.0 : cA + (sA - offw);               // alpha(j-1, c0-1)
                o[2] = first ? 0.0 : cw0 + le;                       // UL(j-1, c0-1)
                o[3] = first ? 0.0 : cw1 + (le - exd);               // UL(j-1, c0-2)
                o[4] = last ? rf0 - rf_top : cR + (sR - offr);       // URin(j-1, c0+W)
                o[5] = 0.5 * (rf0 + rf1);                            // row-total average
            }
            cA += __shfl_sync(FULL, sA, 31);
            cL += __shfl_sync(FULL, sL, 31);
            cR += __shfl_sync(FULL, sR, 31);
        }
    }
    A ul[CPT], al[CPT], cc[CPT], ur[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        al[k] = D.csX[bb * n + x];
        ul[k] = D.dgXc[bb * n + x];
        const double cfi = csT[x], cfe = x > 0 ? csT[x - 1] : 0.0;
        cc[k] = 0.5 * (cfe + cfi);
        ur[k] = 0.0;
    }
    const A Cr = rowfull[n];
    const double inv_nd = 1.0 / (double)n;  // exact: n is a power of two
    const A inv_n = inv_nd;
    const A inv2m = 0.5 * inv_nd * inv_nd;
    const A xc0 = ((double)x0 + 0.5) * inv_nd;  // pixel-centre x of column x0 (displacement.py:59)
    const A hC = 0.5 * Cr;
    const bool zero0 = x0 == 0;
    // ---- the warp's label ring (KP = 4 slots of W ints; row r sits in slot r & 3) ----
    int* rq = align16(s_lut + (LUTS ? lut_smem_len(R) : 0)) + wl * KP * W;
    const unsigned rq_s = (unsigned)__cvta_generic_to_shared(rq);
    const unsigned bar_s = (unsigned)__cvta_generic_to_shared(s_bar + wl * KP);
    const int* glab = D.labels + (size_t)b * D.nn + (size_t)jt * n + c0;  // row jt of the slice
    constexpr int PF = DET_SAT3X_PIPE == 1 ? KP : KP - 1;  // rows fetched by the prologue
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < KP; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s + 8u * s));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
        for (int p = 0; p < PF; ++p)
            if (p < H) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s + 8u * p), "r"(W * 4)
                             : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
                                 "r"(rq_s + (unsigned)(p * W * 4)), "l"(glab + (size_t)p * n), "r"(W * 4), "r"(bar_s + 8u * p)
                             : "memory");
            }
    }
    const int* gnext = glab + (size_t)PF * n;  // the row the next refill fetches
    __syncthreads();  // windows, LUT and (for its own warp) records published: the only CTA barrier

    const A2* pdt = win_dt + ((c0 - cb) >> 2) + lane;
    const A* ptv = win_tv + ((c0 - cb) >> 2) + lane + Hq;
    const A2* prec = reinterpret_cast<const A2*>(s_rec + (size_t)wl * H * 6);
    const int* rsrc = rq + lane * CPT;
    double* o = reinterpret_cast<double*>(D.uf) + (size_t)b * D.nn * 2 + ((size_t)jt * n + x0) * 2;
    const size_t ostep = (size_t)n * 2;
    A yc = ((double)jt + 0.5) * inv_nd;  // (j + 0.5) / n, advanced exactly by 1/n per row
    int rows_left = H;                   // rows from this one to the band end
    unsigned parity = 0;

    // labels in ring slot SL (phase parity par) -> residual densities and the lane's exclusive
    // in-slice row prefix
    A rho_n[CPT], pre_n = 0.0;
    auto take = [&](auto sl_c, unsigned par) {
        constexpr int SL = decltype(sl_c)::value;
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(bar_s + 8u * SL), "r"(par)
                : "memory");
        }
        const int4 Lv = *reinterpret_cast<const int4*>(rsrc + SL * W);
        rho_n[0] = LUTS ? lut[Lv.x] : lut[Lv.x < 0 ? R : Lv.x];
        rho_n[1] = LUTS ? lut[Lv.y] : lut[Lv.y < 0 ? R : Lv.y];
        rho_n[2] = LUTS ? lut[Lv.z] : lut[Lv.z < 0 ? R : Lv.z];
        rho_n[3] = LUTS ? lut[Lv.w] : lut[Lv.w < 0 ? R : Lv.w];
        const A tsum = ((rho_n[0] + rho_n[1]) + rho_n[2]) + rho_n[3];
        pre_n = warp_incl_scan_t<A>(tsum) - tsum;
    };
    if (DET_SAT3X_PIPE) take(std::integral_constant<int, 0>{}, 0u);

    auto row = [&](auto rr_c) {
        constexpr int RR = decltype(rr_c)::value;
        // ---- labels -> residual densities; refill a consumed slot ----
        __syncwarp();
        if (lane == 0 && rows_left > PF) {
            // PIPE: row r's slot (read one row ago) takes row r + 4; else row r-1's slot takes row r + 3
            constexpr int SL = DET_SAT3X_PIPE == 1 ? RR : ((RR + KP - 1) & 3);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s + 8u * SL), "r"(W * 4)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
                             "r"(rq_s + (unsigned)(SL * W * 4)), "l"(gnext), "r"(W * 4), "r"(bar_s + 8u * SL)
                         : "memory");
        }
        gnext += n;
        A rho[CPT], pre;
        if (DET_SAT3X_PIPE == 2) {
            // the NEXT row's labels -> row-prefix scan first (only the prefix is carried over), then
            // this row's densities re-read from its slot: the scan's shuffle chain overlaps this
            // row's field arithmetic at the cost of one more label / LUT read per pixel
            pre = pre_n;
            if (rows_left > 1) take(std::integral_constant<int, (RR + 1) & 3>{}, RR == 3 ? parity ^ 1u : parity);
            const int4 Lv = *reinterpret_cast<const int4*>(rsrc + RR * W);
            rho[0] = LUTS ? lut[Lv.x] : lut[Lv.x < 0 ? R : Lv.x];
            rho[1] = LUTS ? lut[Lv.y] : lut[Lv.y < 0 ? R : Lv.y];
            rho[2] = LUTS ? lut[Lv.z] : lut[Lv.z < 0 ? R : Lv.z];
            rho[3] = LUTS ? lut[Lv.w] : lut[Lv.w < 0 ? R : Lv.w];
        } else if (DET_SAT3X_PIPE == 1) {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
            pre = pre_n;
            if (rows_left > 1) take(std::integral_constant<int, (RR + 1) & 3>{}, RR == 3 ? parity ^ 1u : parity);
        } else {
            take(rr_c, parity);
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
            pre = pre_n;
        }
        --rows_left;
        // ---- edge record of the row (broadcast loads) ----
        const A2 e01 = prec[RR * 3 + 0], e23 = prec[RR * 3 + 1], e45 = prec[RR * 3 + 2];
        A loc[CPT];
        A run = 0.0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) { run += rho[k]; loc[k] = run; }
        const A excl = e01.x + pre;
        A ap_m1 = __shfl_up_sync(FULL, al[CPT - 1], 1);
        A ul_m1 = __shfl_up_sync(FULL, ul[CPT - 1], 1);
        A ul_m2 = __shfl_up_sync(FULL, ul[CPT - 2], 1);
        A ur_p = __shfl_down_sync(FULL, ur[0], 1);
        if (lane == 0) { ap_m1 = e01.y; ul_m1 = e23.x; ul_m2 = e23.y; }
        if (lane == 31) ur_p = e45.x;
        A Av[CPT], an[CPT], uln[CPT], urn[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) Av[k] = excl + loc[k];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            an[k] = al[k] + Av[k];
            uln[k] = Av[k] + (k == 0 ? ul_m1 : ul[k - 1]);
            urn[k] = Av[k] + (k == CPT - 1 ? ur_p : ur[k + 1]);
        }
        const A ravg = e45.y;
        const A ycm1 = yc - 1.0, c1y = 0.25 - 0.5 * yc;
        const A hravg = 0.5 * ravg;
        A dlw[CPT + 1], tuw[CPT], tvw[CPT];
#pragma unroll
        for (int q = 0; q <= CPT; ++q) {
            const A2 v = pdt[((RR + q) & 3) * P + ((RR + q) >> 2)];
            dlw[q] = v.x;
            if (q < CPT) tuw[q] = v.y;
        }
#pragma unroll
        for (int k = 0; k < CPT; ++k) tvw[k] = ptv[((3 - RR + k) & 3) * P + ((3 - RR + k) >> 2)];
        A ux[CPT], uy[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const A apm1 = k == 0 ? ap_m1 : al[k - 1];
            const A anm1 = k == 0 ? (ap_m1 + excl) : an[k - 1];
            const A ulnm1 = k == 0 ? (excl + ul_m2) : uln[k - 1];
            const A ulpm1 = k == 0 ? ul_m1 : ul[k - 1];
            const A ulpm2 = k == 0 ? ul_m2 : (k == 1 ? ul_m1 : ul[k - 2]);
            const A urp1 = k == CPT - 1 ? ur_p : ur[k + 1];
            const A Dw = dlw[k + 1], Dwm1 = dlw[k];
            const A R_UV = ulpm1 + (Dw - urp1);
            A R_UVm1 = ulnm1 + (Dw - urn[k]);
            A R_Um1Vm1 = ulpm2 + (Dwm1 - ur[k]);
            if (k == 0 && zero0) { R_UVm1 = 0.0; R_Um1Vm1 = 0.0; }
            const A bt = R_UVm1;
            const A at = tuw[k] - R_Um1Vm1 + rho[k];
            const A gt = tvw[k] - R_UV;
            // branch-free anchor combination (see k_sat3, DET_SAT3_ABS)
            const A a4 = apm1 + al[k] + anm1 + an[k];  // 4a
            const A cavg = cc[k];
            const A xc = xc0 + (A)k * inv_n;
            const A e = xc + ycm1, d = xc - yc;
            const A ae = fabs(e), ad = fabs(d);
            const A hs = fma(0.5, cavg, hravg), hd = fma(-0.5, cavg, hravg);
            const A hK = hs - hC;
            const A tt = at + gt;
            A vx = fma(a4, c1y, cavg);
            vx = fma(hs, e, vx);
            vx = fma(hd, ae, vx);
            vx = fma(-hK, d + ad, vx);
            vx = fma(xc, tt, vx);
            ux[k] = (vx + bt) * inv2m;
            A vy = fma(a4, fma(xc, -0.5, 0.25), ravg);
            vy = fma(hs, e, vy);
            vy = fma(-hd, ae, vy);
            vy = fma(hK, d - ad, vy);
            vy = fma(yc, Cr - tt, vy);
            uy[k] = (vy + at) * inv2m;
        }
#pragma unroll
        for (int k = 0; k < CPT; k += 2)
#ifdef DET_SAT3X_SKIPTEST  // timing experiment only (invalid field): half of the sector stores dropped
            if (((RR + lane + (k >> 1)) & 1) == 0)
#endif
            st_global_v4f64(o + 2 * k, ux[k], uy[k], ux[k + 1], uy[k + 1]);
        o += ostep;
        yc += inv_n;
#pragma unroll
        for (int k = 0; k < CPT; ++k) { al[k] = an[k]; ul[k] = uln[k]; ur[k] = urn[k]; }
    };

    int r = 0;
    for (; r + 4 <= H; r += 4) {
        row(std::integral_constant<int, 0>{});
        row(std::integral_constant<int, 1>{});
        row(std::integral_constant<int, 2>{});
        row(std::integral_constant<int, 3>{});
        pdt += 1;
        ptv -= 1;
        prec += 12;
        parity ^= 1u;
    }
    if (r < H) {  // band heights that are not a multiple of four
        row(std::integral_constant<int, 0>{});
        if (r + 1 < H) row(std::integral_constant<int, 1>{});
        if (r + 2 < H) row(std::integral_constant<int, 2>{});
    }
    if constexpr (FA) {
        if (fa_par >= 0) {
            __syncthreads();  // every warp's rows of the band are written; windows and records are dead
            advect_band_vertices(D, b, band, fa_par, wl, NWC, lane, reinterpret_cast<int*>(s_raw3x) + wl * 512, uq_off);
        }
    }
}

// ---------------------------------------------------------------------------------
// k_sat1x: k_sat1w<4, NT, LUTS, double, TAB> (the float64 field's band sums and slice tables) with the
// row loop unrolled four times over an 8-slot warp ring (two halves of four compile-time slots,
// prefetch distance 6 rows), the slice exports written through advancing pointers, and the band-end
// dg / ad staging aliased onto the ring and LUT area (free once the sweep is over).  Same sums in
// the same order as k_sat1w.
#ifndef DET_SAT1X_MINB
#define DET_SAT1X_MINB 2  // 90 registers, no spill (3 CTAs/SM at 80 registers spills: 46.9k vs 51.7k it/s)
#endif
template <int NT, bool LUTS>
__global__ void __launch_bounds__(NT, (NT <= 256 ? DET_SAT1X_MINB : 1)) k_sat1x(Topo T, Bufs D, int gate) {
    using A = double;
    constexpr int CPT = 4, NW = NT / 32, W = 32 * CPT, KP = 8;
    // row partials [H][NW] | exitD [NW][H] | exitA [NW][H] | E1 [NW][H] | { rings, LUT } aliased by { dg[L] | ad[L] }
    extern __shared__ __align__(16) unsigned char s_raw1x[];
    __shared__ uint64_t s_bar[NW * KP];
    __shared__ double s_red[33];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, L = n + H - 1, R = T.R;
    const int x0 = t * CPT, c0 = w * W;
    const size_t bb = (size_t)b * D.nb + band;
    A* s_rows = reinterpret_cast<A*>(s_raw1x);
    A* exD = s_rows + H * NW;
    A* exA = exD + NW * H;
    A* exE = exA + NW * H;
    int* ring_base = reinterpret_cast<int*>(exE + NW * H);  // 16-byte aligned: 4*H*NW doubles
    A* s_lut = reinterpret_cast<A*>(ring_base + NW * KP * W);
    A* dg = reinterpret_cast<A*>(ring_base);                // band end only
    A* ad = dg + L;
    const A* glut = reinterpret_cast<const A*>(D.lut + (size_t)b * (R + 1));
    if (LUTS)  // background-first (see band_lut): labels index s_lut + 1 directly
        for (int i = t; i <= R; i += NT) s_lut[i] = __ldg(glut + (i == 0 ? R : i - 1));
    const A* lut = LUTS ? s_lut + 1 : glut;
    int* rq = ring_base + w * KP * W;
    const unsigned rq_s = (unsigned)__cvta_generic_to_shared(rq);
    const unsigned bar_s = (unsigned)__cvta_generic_to_shared(s_bar + w * KP);
    const int* glab = D.labels + (size_t)b * D.nn + (size_t)jt * n + c0;
    auto fetch = [&](const int* src, unsigned slot) {  // lane 0: one 512-byte slice row into a slot
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s + 8u * slot), "r"(W * 4)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
                         "r"(rq_s + slot * (unsigned)(W * 4)), "l"(src), "r"(W * 4), "r"(bar_s + 8u * slot)
                     : "memory");
    };
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < KP; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s + 8u * s));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
        for (int p = 0; p < KP - 1; ++p)
            if (p < H) fetch(glab + (size_t)p * n, (unsigned)p);
    }
    __syncwarp();
    if (LUTS) __syncthreads();  // LUT published

    A cs[CPT], pd[CPT], pa[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) cs[k] = pd[k] = pa[k] = 0.0;
    A rho_n[CPT];
    const int* gnext = glab + (size_t)(KP - 1) * n;  // the row the next refill fetches
    int fetch_left = H - (KP - 1);                   // rows still to fetch
    unsigned half = 0, parity = 0;                   // ring half (slots 4*half ..), its phase parity
    const int* rsrc = rq + lane * CPT;
    A* pxd = exD + w * H;
    A* pxa = exA + w * H;
    A* prow = s_rows + w;

    // labels of the row in slot SL of ring half hf -> rho_n (waits for the slot's copy)
    auto take = [&](auto sl_c, unsigned hf, unsigned par) {
        constexpr int SL = decltype(sl_c)::value;
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(bar_s + 8u * SL + 32u * hf), "r"(par)
                : "memory");
        }
        const int4 Lv = *reinterpret_cast<const int4*>(rsrc + SL * W + hf * (4 * W));
        rho_n[0] = LUTS ? lut[Lv.x] : __ldg(lut + (Lv.x < 0 ? R : Lv.x));
        rho_n[1] = LUTS ? lut[Lv.y] : __ldg(lut + (Lv.y < 0 ? R : Lv.y));
        rho_n[2] = LUTS ? lut[Lv.z] : __ldg(lut + (Lv.z < 0 ? R : Lv.z));
        rho_n[3] = LUTS ? lut[Lv.w] : __ldg(lut + (Lv.w < 0 ? R : Lv.w));
    };
    take(std::integral_constant<int, 0>{}, 0u, 0u);

    // Slice row totals of four rows in one butterfly: the half-warps take rows {0,1} / {2,3}, the
    // quarter-warps one row of the pair, then three steps inside each group of eight lanes -- 6
    // double shuffles in 5 dependent steps for 4 sums (lanes 0, 8, 16, 24 end with them).  Issued
    // inside the NEXT group's first row, so its shuffle chain overlaps that row's arithmetic.
    // E1 (the slice's sum of a row's diagonal partials) needs no per-lane work: summing the
    // recurrence pd(r, x) = rho(r, x) + pd(r-1, x-1) over the slice gives
    //   E1(r) = total(r) + E1(r-1) - pd(r-1, last column) = sum_{r'<=r} total(r') - sum_{r'<r} exitD(r'),
    // two warp scans per slice at the band end.
    A tsv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) tsv[q] = 0.0;
    auto flush4 = [&](A* prow_g, int nv) {
        const bool b4 = (lane & 16) != 0, b3 = (lane & 8) != 0;
        const A k0 = (b4 ? tsv[2] : tsv[0]) + __shfl_xor_sync(FULL, b4 ? tsv[0] : tsv[2], 16);
        const A k1 = (b4 ? tsv[3] : tsv[1]) + __shfl_xor_sync(FULL, b4 ? tsv[1] : tsv[3], 16);
        A v = (b3 ? k1 : k0) + __shfl_xor_sync(FULL, b3 ? k0 : k1, 8);
        v += __shfl_xor_sync(FULL, v, 4);
        v += __shfl_xor_sync(FULL, v, 2);
        v += __shfl_xor_sync(FULL, v, 1);
        const int row = ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
        if ((lane & 7) == 0 && row < nv) prow_g[row * NW] = v;
    };
    // one band row; RR = r & 3, `more`: a next row exists (its labels are taken one row early);
    // `flush`: the previous group's four row sums are reduced here
    auto row = [&](auto rr_c, bool more, bool flush) {
        constexpr int RR = decltype(rr_c)::value;
        A rho[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
        // the slot of row r-1 (read one row ago by every lane) takes row r + KP - 1
        __syncwarp();
        if (lane == 0 && fetch_left > 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            fetch(gnext, (unsigned)((RR + 3) & 3) + 4u * (RR == 0 ? (half ^ 1u) : half));
        }
        gnext += n;
        --fetch_left;
        if (more) {
            if constexpr (RR == 3) take(std::integral_constant<int, 0>{}, half ^ 1u, half ? parity ^ 1u : parity);
            else take(std::integral_constant<int, RR + 1>{}, half, parity);
        }
        if (RR == 0 && flush) flush4(prow - 4 * NW, 4);
        A ts = 0.0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) ts += rho[k];
        A left = __shfl_up_sync(FULL, pd[CPT - 1], 1);
        A right = __shfl_down_sync(FULL, pa[0], 1);
        if (lane == 0) left = 0.0;    // partials restart at the slice edge
        if (lane == 31) right = 0.0;
#pragma unroll
        for (int k = CPT - 1; k >= 0; --k) pd[k] = rho[k] + (k == 0 ? left : pd[k - 1]);
#pragma unroll
        for (int k = 0; k < CPT; ++k) pa[k] = rho[k] + (k == CPT - 1 ? right : pa[k + 1]);
#pragma unroll
        for (int k = 0; k < CPT; ++k) cs[k] += rho[k];
        if (lane == 31) pxd[RR] = pd[CPT - 1];  // diagonal leaving the slice's right edge
        if (lane == 0) pxa[RR] = pa[0];         // anti-diagonal leaving the slice's left edge
        tsv[RR] = ts;
    };
    int r = 0;
    for (; r + 4 <= H; r += 4) {
        const bool more = r + 4 < H;
        row(std::integral_constant<int, 0>{}, true, r > 0);
        row(std::integral_constant<int, 1>{}, true, false);
        row(std::integral_constant<int, 2>{}, true, false);
        row(std::integral_constant<int, 3>{}, more, false);
        pxd += 4; pxa += 4; prow += 4 * NW;
        if (half) parity ^= 1u;
        half ^= 1u;
    }
    if (r > 0) {
        flush4(prow - 4 * NW, 4);
    } else {  // band heights 1 and 2
        row(std::integral_constant<int, 0>{}, H > 1, false);
        if (H > 1) row(std::integral_constant<int, 1>{}, false, false);
        flush4(prow, H);
    }
    __syncthreads();  // exits, row partials published; ring and LUT free (dg / ad alias them)
    {   // E1 of this warp's slice from its row totals and diagonal exits (published by the barriers below)
        A ct = 0.0, cd = 0.0;
        for (int r0 = 0; r0 < H; r0 += 32) {
            const int rr = r0 + lane;
            const A tv = rr < H ? s_rows[rr * NW + w] : 0.0, dv = rr < H ? exD[w * H + rr] : 0.0;
            const A st = warp_incl_scan_t<A>(tv), sd = warp_incl_scan_t<A>(dv);
            if (rr < H) exE[w * H + rr] = (ct + st) - (cd + (sd - dv));
            ct += __shfl_sync(FULL, st, 31);
            cd += __shfl_sync(FULL, sd, 31);
        }
    }
    // band-bottom entries + the neighbour slice's part of each crossing diagonal
    double csum = 0.0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        const int xi = x - c0;                       // column inside the slice
        A vd = pd[k], va = pa[k];
        if (w > 0 && xi <= H - 2) vd += exD[(w - 1) * H + (H - 2 - xi)];
        const int xr = W - 1 - xi;                   // columns to the slice's right edge
        if (w < NW - 1 && xr <= H - 2) va += exA[(w + 1) * H + (H - 2 - xr)];
        dg[x] = vd;
        ad[H - 1 + x] = va;
        csum += cs[k];
    }
    // diagonals leaving the texture's right edge / anti-diagonals leaving its left edge (j < jb)
    if (t < H - 1) {
        dg[n - 1 - (jt + t) + jb] = exD[(NW - 1) * H + t];
        ad[t] = exA[t];
    }
    double tot;
    double run = block_excl_scan(csum, s_red, &tot);  // (its barriers also publish dg/ad)
    double* tab = D.tab + bb * 4 * NW * H;
    if (t < H) {  // row totals in float64, warp order
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            tab[q * H + t] = s;  // off(t, q): the slice totals left of slice q
            s += s_rows[t * NW + q];
        }
        D.rt[(size_t)b * n + jt + t] = s;
    }
    for (int i = t; i < NW * H; i += NT) {
        tab[NW * H + i] = exE[i];
        tab[2 * NW * H + i] = exD[i];
        tab[3 * NW * H + i] = exA[i];
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        run += cs[k];
        D.cs[bb * n + x0 + k] = run;
    }
    block_prefix_smem<A>(dg, D.dgc + bb * L, L, s_red);
    block_prefix_smem<A>(ad, D.adc + bb * L, L, s_red);
}

}  // namespace det
