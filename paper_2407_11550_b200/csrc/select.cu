// select.cu -- K2/K3 selection: layer-wide radix select -> adaptive budgets ->
// safeguard/repair -> per-segment radix select -> keep mask + kept positions.
//
// Replaces adaptive_allocation (budget.hpp:118-140: layer-wide top-`total` over the
// concatenated segments, ordered (score desc, head asc, pos asc) = flat order),
// safeguard_blend + apportion (145-158, 45-93), uniform_allocation (103-113),
// repair_zero_budgets (policies.hpp:178-196), topk_decision (80-93: ties to the
// lowest position) and streaming_llm_decision (159-165).
//
// Design (B200): one thread-block cluster of CS <= 8 CTAs per problem, 1024
// threads each; CTA r owns a contiguous slice of the problem's flattened scores.
// Keys are the scores' bit patterns mapped to an order-preserving unsigned integer
// (-0 canonicalised to +0), selected MSB-first with 8-bit digits: per-CTA
// per-segment shared-memory histograms (warp-aggregated with match.any), summed
// across the cluster through distributed shared memory, one cluster barrier per
// digit (double-buffered histograms).  Exactness: the threshold key T and the
// number of T-equal elements to take are integers, and "lowest flat index wins a
// tie" is realised by ballot-ranked prefix counts in flat order, so budgets, keep
// masks and kept positions are bit-identical to the reference on identical scores.
#include <cooperative_groups.h>

#include <map>
#include <mutex>
#include <tuple>

#include "select.cuh"

namespace cg = cooperative_groups;

namespace adakv_b200 {



// (debug) per-CTA clock64 stamps of the select phases (ADAKV debug hook, scripts only)
static unsigned long long* g_sel_dbg = nullptr;

namespace {

constexpr int kSelThreads = 1024;
constexpr int kWarps = kSelThreads / 32;
constexpr int kEChunks = 8;  // phase E: 32-key chunks per warp with their loads in flight
constexpr int kMaxSelCS = 16;  // CTAs per cluster (16 needs the non-portable cluster size)

enum SegMode : int { MODE_NONE = 0, MODE_ALL = 1, MODE_THRESH = 2, MODE_STREAM = 3 };

template <class F> struct KeyOf;
template <> struct KeyOf<float> {
    using type = uint32_t;
    static constexpr int kBits = 32;
    __device__ static uint32_t get(float x) {
        uint32_t b = __float_as_uint(x);
        if (b == 0x80000000u) b = 0u;  // -0 == +0 (the reference compares with !=, >)
        return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    }
    __device__ static uint32_t bits(float x) { return __float_as_uint(x); }
};
template <> struct KeyOf<double> {
    using type = unsigned long long;
    static constexpr int kBits = 64;
    __device__ static unsigned long long get(double x) {
        unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
        if (b == 0x8000000000000000ull) b = 0ull;
        return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
    }
    __device__ static unsigned long long bits(double x) { return static_cast<unsigned long long>(__double_as_longlong(x)); }
};

struct BinPick {
    int bin;
    int64_t cum_above;
};

// Warp-cooperative: in a 256-bin histogram find the bin holding the krem-th
// largest element (krem >= 1), scanning bins from high to low.
__device__ __forceinline__ BinPick find_bin(const uint32_t* h, int64_t krem, int lane) {
    int64_t s8 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s8 += h[lane * 8 + i];
    int64_t suf = s8;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf += t;
    }
    int64_t next = __shfl_down_sync(0xffffffffu, suf, 1);
    if (lane == 31) next = 0;
    const unsigned hit = __ballot_sync(0xffffffffu, suf >= krem && next < krem);
    const int L = hit ? __ffs(hit) - 1 : 0;
    int bin = 0;
    int64_t cum = 0;
    if (lane == L) {
        cum = next;
        bin = L * 8;
        for (int i = 7; i >= 0; --i) {
            const int64_t c = h[L * 8 + i];
            if (cum + c >= krem) {
                bin = L * 8 + i;
                break;
            }
            cum += c;
        }
    }
    bin = __shfl_sync(0xffffffffu, bin, L);
    cum = __shfl_sync(0xffffffffu, cum, L);
    return {bin, cum};
}

// NONNEG: all scores are +0 or positive (SelParams::nonneg), so a score's bit pattern already
// orders as its value and the order-preserving key transform is skipped (~20% of the scans)
template <class F, bool NONNEG>
__global__ void __launch_bounds__(kSelThreads, 1) select_kernel(const SelParams prm, unsigned long long* dbg) {
    using KT = typename KeyOf<F>::type;
    constexpr int kBits = KeyOf<F>::kBits;
    auto kget = [](F x) -> KT {
        if constexpr (NONNEG) return KeyOf<F>::bits(x);
        else return KeyOf<F>::get(x);
    };
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned CS = cluster.num_blocks();
    const unsigned rank = cluster.block_rank();
    const int64_t p = blockIdx.x / CS;
    const int S = prm.S;
    const int64_t N = prm.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const F* sc = static_cast<const F*>(prm.scores) + p * N;
    const int64_t lo = N * rank / CS, hi = N * (rank + 1) / CS;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const bool lean = prm.lean != 0;
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw);     // [2][S][256] ([1] when lean)
    uint32_t* agg = hist + (lean ? 1 : 2) * S * 256;             // [S][256]
    uint32_t* hist0 = agg + S * 256;                             // [S][256] (none when lean)
    uint32_t* wcnt = hist0 + (lean ? 0 : S * 256);               // [kWarps][S][2]
    int64_t* wkept = reinterpret_cast<int64_t*>(wcnt + kWarps * S * 2);  // [kWarps][S]
    int64_t* weqb = wkept + kWarps * S;                                  // [kWarps][S]
    uint32_t* wh = reinterpret_cast<uint32_t*>(weqb + kWarps * S);       // [kWarps][256] per-warp histograms
    KT* kc = reinterpret_cast<KT*>(wh + kWarps * 256);                   // [hi - lo] cached keys

    __shared__ uint32_t ccnt[kMaxSeg][2];  // this CTA's (gt, eq) per segment
    __shared__ KT seg_prefix[kMaxSeg];
    __shared__ int64_t seg_krem[kMaxSeg], seg_gt[kMaxSeg], seg_need[kMaxSeg];
    __shared__ KT seg_T[kMaxSeg];
    __shared__ int seg_mode[kMaxSeg], seg_active[kMaxSeg];
    __shared__ int64_t seg_sink[kMaxSeg], seg_recent[kMaxSeg], seg_eqb[kMaxSeg];
    __shared__ uint64_t b_raw[kMaxSeg], b_fin[kMaxSeg], b_caps[kMaxSeg];
    __shared__ double quotas[kMaxSeg];
    __shared__ int64_t wkept_before[kWarps];
    __shared__ KT g_T, g_common;
    __shared__ int64_t g_take, g_k;
    __shared__ int any_active, have_hist0;
    __shared__ uint32_t s_err;

    int nst = 0;
    auto stamp = [&]() {
        if (dbg && tid == 0 && nst < 24) dbg[blockIdx.x * 32 + nst] = clock64();
        ++nst;
    };
    int fine_pass = -1;  // (debug) fine stamps of one radix pass into slots 24..31
    auto fstamp = [&](int k) {
        if (dbg && tid == 0 && fine_pass == 1) dbg[blockIdx.x * 32 + 24 + k] = clock64();
    };
    stamp();
    if (tid == 0) {
        s_err = 0;
        have_hist0 = 0;
        g_k = prm.totals ? prm.totals[p] : prm.total;
    }
    // segment tables read by every pass: offsets, the ranks holding each segment's elements
    // (the only ranks whose histograms the DSMEM sum reads) and this CTA's segment range
    __shared__ int64_t s_off[kMaxSeg + 1];
    __shared__ unsigned char seg_r0[kMaxSeg], seg_r1[kMaxSeg];
    __shared__ int c_s0, c_s1;
    for (int s = tid; s <= S; s += kSelThreads) s_off[s] = prm.off[s];
    // rank owning flat element e: the exact inverse of the slice split above (CTA t owns
    // [N t / CS, N (t+1) / CS)), i.e. the largest t with floor(N t / CS) <= e
    auto rank_of = [&](int64_t e) -> unsigned {
        unsigned r = 0;
        for (unsigned t = 1; t < CS; ++t)
            if (N * int64_t(t) / int64_t(CS) <= e) r = t;
        return r;
    };
    for (int s = tid; s < S; s += kSelThreads) {
        seg_gt[s] = 0;
        b_caps[s] = uint64_t(prm.off[s + 1] - prm.off[s]);
        seg_r0[s] = (unsigned char)rank_of(prm.off[s]);
        seg_r1[s] = (unsigned char)rank_of(prm.off[s + 1] > 0 ? prm.off[s + 1] - 1 : 0);
    }

    // Every pass below re-reads this CTA's slice of keys: read the scores from global memory
    // once, in coalesced order, and keep the order-preserving keys in shared memory.
    const bool cached = prm.cache_keys != 0;
    if (cached) {
        // 16-byte loads, four in flight per thread (scalar head up to the first aligned element)
        constexpr int V = 16 / int(sizeof(F));
        const F* src = sc + lo;
        const int64_t len = hi - lo;
        const int64_t mis = int64_t(reinterpret_cast<uintptr_t>(src) / sizeof(F)) % V;
        const int64_t h0 = min(len, (V - mis) % V);
        for (int64_t i = tid; i < h0; i += kSelThreads) kc[i] = kget(src[i]);
        const int64_t nv = (len - h0) / V;
        const uint4* vs = reinterpret_cast<const uint4*>(src + h0);
        for (int64_t t0 = tid; t0 < nv; t0 += 4 * kSelThreads) {
            uint4 r[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t t = t0 + int64_t(u) * kSelThreads;
                r[u] = t < nv ? __ldcs(vs + t) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t t = t0 + int64_t(u) * kSelThreads;
                if (t >= nv) break;
                const F* f = reinterpret_cast<const F*>(&r[u]);
                KT kk[V];
#pragma unroll
                for (int c = 0; c < V; ++c) kk[c] = kget(f[c]);
                if (h0 == 0) {
                    *reinterpret_cast<uint4*>(kc + t * V) = *reinterpret_cast<const uint4*>(kk);
                } else {
#pragma unroll
                    for (int c = 0; c < V; ++c) kc[h0 + t * V + c] = kk[c];
                }
            }
        }
        for (int64_t i = h0 + nv * V + tid; i < len; i += kSelThreads) kc[i] = kget(src[i]);
    }
    auto key_at = [&](int64_t e) -> KT { return cached ? kc[e - lo] : kget(sc[e]); };
    // Uncached slices (too large for shared memory): every key of [a, b) from global memory
    // (L2) through fn(e, key), 16-byte loads with four per thread in flight; the unaligned
    // head and tail elements are read singly so no load leaves [a, b).
    auto scan_global = [&](int64_t a, int64_t b, auto&& fn) {
        constexpr int V = 16 / int(sizeof(F));
        const int64_t mis = int64_t(reinterpret_cast<uintptr_t>(sc + a) / sizeof(F)) % V;
        const int64_t va = min(b, a + (V - mis) % V);  // first vector-aligned element
        const int64_t nv = (b - va) / V;
        const int64_t vb = va + nv * V;
        for (int64_t e = a + tid; e < va; e += kSelThreads) fn(e, kget(sc[e]));
        for (int64_t e = vb + tid; e < b; e += kSelThreads) fn(e, kget(sc[e]));
        const uint4* vs = reinterpret_cast<const uint4*>(sc + va);
        for (int64_t t0 = tid; t0 < nv; t0 += 4 * kSelThreads) {
            uint4 r[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t t = t0 + int64_t(u) * kSelThreads;
                r[u] = t < nv ? __ldcg(vs + t) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t t = t0 + int64_t(u) * kSelThreads;
                if (t >= nv) break;
                const F* f = reinterpret_cast<const F*>(&r[u]);
#pragma unroll
                for (int c = 0; c < V; ++c) fn(va + t * V + c, kget(f[c]));
            }
        }
    };
    __syncthreads();
    stamp();
    if (tid == 0) {
        // the segments whose DSMEM sum reads this rank's histograms (the same rank ranges as
        // the sum uses, so an empty segment at a slice boundary is covered too); published
        // by the barriers of the min/max step below
        int s0 = S, s1 = -1;
        for (int s = 0; s < S; ++s)
            if (seg_r0[s] <= rank && rank <= seg_r1[s]) {
                s0 = s < s0 ? s : s0;
                s1 = s;
            }
        c_s0 = s0;
        c_s1 = s1;
    }

    // Bits shared by every key of the problem are skipped: the radix digits start at the
    // highest bit where the problem's min and max keys differ.  (Scores concentrate in a
    // few exponent values, so a digit over the raw top byte would put most keys in a
    // handful of bins and serialise the histogram atomics.)
    __shared__ KT red_mm[kWarps][2];
    __shared__ KT cta_mm[2];
    __shared__ int s_top;
    {
        KT mn = ~KT(0), mx = KT(0);
        auto fold = [&](int64_t, KT u) {
            mn = u < mn ? u : mn;
            mx = u > mx ? u : mx;
        };
        if (cached)
            for (int64_t e = lo + tid; e < hi; e += kSelThreads) fold(e, kc[e - lo]);
        else
            scan_global(lo, hi, fold);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const KT a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
        }
        if (lane == 0) {
            red_mm[warp][0] = mn;
            red_mm[warp][1] = mx;
        }
        __syncthreads();
        if (tid == 0) {
            KT a = ~KT(0), b = KT(0);
            for (int w = 0; w < kWarps; ++w) {
                a = red_mm[w][0] < a ? red_mm[w][0] : a;
                b = red_mm[w][1] > b ? red_mm[w][1] : b;
            }
            cta_mm[0] = a;
            cta_mm[1] = b;
        }
        cluster.sync();
        if (tid == 0) {
            KT a = ~KT(0), b = KT(0);
            for (int rb = 0; rb < int(CS); rb += 8) {
                KT v[2][8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    v[0][r] = unsigned(rb + r) < CS ? cluster.map_shared_rank(cta_mm, rb + r)[0] : ~KT(0);
                    v[1][r] = unsigned(rb + r) < CS ? cluster.map_shared_rank(cta_mm, rb + r)[1] : KT(0);
                }
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    a = v[0][r] < a ? v[0][r] : a;
                    b = v[1][r] > b ? v[1][r] : b;
                }
            }
            // empty problem slices leave a > b; any top works then
            const KT x = a <= b ? (a ^ b) : KT(0);
            s_top = x == 0 ? 0 : kBits - (kBits == 32 ? __clz(uint32_t(x)) : __clzll((long long)x));
            g_common = a <= b ? a : KT(0);
        }
        __syncthreads();
    }
    const int top = s_top;                              // significant low bits
    const int npass = top == 0 ? 1 : (top + 7) / 8;     // radix passes
    auto lo_bit = [&](int pass) { const int v = top - 8 * (pass + 1); return v < 0 ? 0 : v; };
    auto hi_mask = [&](int pass) {                     // bits above this pass's digit
        const int hb = top - 8 * pass;
        return hb >= kBits ? KT(0) : (~KT(0)) << hb;
    };
    const KT common = g_common & hi_mask(0);

    // One radix digit over all segments with seg_active[s] set: per-segment
    // histograms of elements matching that segment's prefix, cluster-summed into agg.
    int buf = 0;  // histogram double buffer; toggled only by a pass that used it
    bool hist_used = false;
    auto radix_pass = [&](int pass) {
        fine_pass = pass;
        // one buffer: every rank has finished reading this CTA's previous histograms
        if (lean && hist_used) cluster.sync();
        hist_used = true;
        if (lean) buf = 0;
        fstamp(0);
        const int shift = lo_bit(pass);
        const KT mask = hi_mask(pass);
        uint32_t* hb = hist + buf * S * 256;
        uint32_t* my = wh + warp * 256;  // this warp's private histogram (no inter-warp atomics)
        // only segments overlapping this CTA's slice: no other rank's DSMEM sum reads the rest
        for (int s = c_s0; s <= c_s1; ++s) {
            const int64_t a = max(lo, s_off[s]), b = min(hi, s_off[s + 1]);
            if (!seg_active[s] || a >= b) {
                for (int i = tid; i < 256; i += kSelThreads) hb[s * 256 + i] = 0;
                continue;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) my[lane * 8 + i] = 0;
            __syncwarp();
            const KT pre = seg_prefix[s];
            if (cached) {
                // 16-byte vector reads of the cached keys: V consecutive keys per thread
                constexpr int V = 16 / int(sizeof(KT));
                // (slice-local indices fit 32 bits; only the vectors straddling the segment
                // ends need per-key range checks)
                const int a0 = int(a - lo), b0 = int(b - lo);
                for (int base = (a0 / V) * V + tid * V; base < b0; base += kSelThreads * V) {
                    const uint4 raw = *reinterpret_cast<const uint4*>(kc + base);
                    const KT* kk = reinterpret_cast<const KT*>(&raw);
                    const bool full = base >= a0 && base + V <= b0;
#pragma unroll
                    for (int i = 0; i < V; ++i) {
                        const KT u = kk[i];
                        const bool in = full || (base + i >= a0 && base + i < b0);
                        if (in && (u & mask) == pre)
                            atomicAdd(&my[int((u >> shift) & 0xFF)], 1u);  // warp-private histogram
                    }
                }
            } else {
                scan_global(a, b, [&](int64_t, KT u) {
                    if ((u & mask) == pre) atomicAdd(&my[int((u >> shift) & 0xFF)], 1u);  // warp-private histogram
                });
            }
            fstamp(1);
            __syncthreads();
            fstamp(2);
            if (tid < 256) {
                uint32_t t = 0;
#pragma unroll 8
                for (int w = 0; w < kWarps; ++w) t += wh[w * 256 + tid];
                hb[s * 256 + tid] = t;
            }
            __syncthreads();
            fstamp(3);
        }
        cluster.sync();
        fstamp(4);
        // sum the CS histograms through DSMEM: all remote loads issued before any is used
        // (segment s has elements only in ranks [r0, r1]: the others' histograms are zero)
        for (int i0 = tid; i0 < S * 256; i0 += 2 * kSelThreads) {
            uint32_t t[2] = {0u, 0u};
            unsigned r0[2], r1[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = i0 + u * kSelThreads;
                const bool in = i < S * 256;
                r0[u] = in ? seg_r0[i >> 8] : 1u;
                r1[u] = in ? seg_r1[i >> 8] : 0u;
            }
            // eight ranks per round (a segment spans more only in clusters of more than 8)
            for (unsigned rb = 0; rb < CS; rb += 8) {
                if (r0[0] + rb > r1[0] && r0[1] + rb > r1[1]) break;
                uint32_t v[2][8];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int i = i0 + u * kSelThreads;
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        v[u][r] = (r0[u] + rb + unsigned(r) <= r1[u]) ? cluster.map_shared_rank(hb, r0[u] + rb + r)[i] : 0u;
                }
#pragma unroll
                for (int u = 0; u < 2; ++u)
                    t[u] += ((v[u][0] + v[u][1]) + (v[u][2] + v[u][3])) + ((v[u][4] + v[u][5]) + (v[u][6] + v[u][7]));
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = i0 + u * kSelThreads;
                if (i < S * 256) agg[i] = t[u];
            }
        }
        fstamp(5);
        __syncthreads();
        fstamp(6);
        buf ^= 1;
        stamp();
    };

    // ---------------- Phase A: layer-wide top-k (Algorithm 1, budget.hpp:118-140)
    const bool adaptive = prm.alloc_mode == ADAKV_ALLOC_ADAPTIVE;
    if (adaptive && g_k > 0 && g_k <= N) {
        __shared__ int64_t g_krem;
        __shared__ KT g_prefix;
        if (tid == 0) {
            g_krem = g_k;
            g_prefix = common;
        }
        for (int s = tid; s < S; s += kSelThreads) seg_active[s] = 1;
        __syncthreads();
        for (int pass = 0; pass < npass; ++pass) {
            for (int s = tid; s < S; s += kSelThreads) seg_prefix[s] = g_prefix;
            __syncthreads();
            radix_pass(pass);
            if (pass == 0) {
                if (!lean) {
                    for (int i = tid; i < S * 256; i += kSelThreads) hist0[i] = agg[i];
                    if (tid == 0) have_hist0 = 1;
                }
            }
            __shared__ int g_bin;
            __shared__ uint32_t gsum[256];
            for (int b = tid; b < 256; b += kSelThreads) {
                uint32_t t = 0;
                for (int s = 0; s < S; ++s) t += agg[s * 256 + b];
                gsum[b] = t;
            }
            __syncthreads();
            if (warp == 0) {
                const BinPick bp = find_bin(gsum, g_krem, lane);
                if (lane == 0) {
                    g_bin = bp.bin;
                    g_krem -= bp.cum_above;
                    g_prefix |= KT(bp.bin) << lo_bit(pass);
                }
            }
            __syncthreads();
            // elements above the chosen bin are definitely selected
            for (int s = warp; s < S; s += kWarps) {
                int64_t t = 0;
                for (int b = g_bin + 1 + lane; b < 256; b += 32) t += agg[s * 256 + b];
                for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (lane == 0) {
                    seg_gt[s] += t;
                    if (pass == npass - 1) seg_need[s] = agg[s * 256 + g_bin];  // eq_s
                }
            }
            __syncthreads();
        }
        if (tid == 0) {
            g_T = g_prefix;
            g_take = g_krem;
            int64_t rem = g_krem;
            for (int s = 0; s < S; ++s) {
                const int64_t take = seg_need[s] < rem ? seg_need[s] : rem;
                rem -= take;
                seg_need[s] = take;  // T-equal elements of segment s inside the layer-wide top-k
                b_raw[s] = uint64_t(seg_gt[s] + take);
            }
        }
    } else if (adaptive && tid == 0) {
        for (int s = 0; s < S; ++s) b_raw[s] = 0;
    }
    __syncthreads();

    stamp();
    // ---------------- Phase C: allocation (one warp, redundantly per CTA, bit-exact fp64)
    if (warp == 0) {
        uint32_t e = 0;
        // a per-problem total outside [0, N] (layer budget below the window floor or above the
        // capacity, policies.hpp:229-231, budget.hpp:48-59) is rejected, never selected from
        if (prm.alloc_mode != ADAKV_ALLOC_GIVEN && (g_k < 0 || g_k > N)) e |= ERR_BUDGET;
        const uint64_t k = e ? 0 : uint64_t(g_k);
        for (int s = lane; s < S; s += 32) b_fin[s] = 0;
        __syncwarp();
        if (e) {
        } else if (adaptive) {
            if (prm.blend) e |= safeguard_warp(b_raw, k, S, prm.alpha, b_caps, quotas, b_fin, lane);
            else
                for (int s = lane; s < S; s += 32) b_fin[s] = b_raw[s];
        } else if (prm.alloc_mode == ADAKV_ALLOC_UNIFORM) {
            e |= uniform_warp(k, S, b_caps, quotas, b_fin, lane);
        } else {
            bool bad = false;
            for (int s = lane; s < S; s += 32) {
                const int64_t b = prm.budgets[p * S + s];
                if (b < 0 || uint64_t(b) > b_caps[s]) bad = true;
                b_fin[s] = b < 0 ? 0 : (uint64_t(b) > b_caps[s] ? b_caps[s] : uint64_t(b));
            }
            if (__any_sync(0xffffffffu, bad)) e |= ERR_BUDGET;
        }
        __syncwarp();
        // repair_zero_budgets only changes anything when a budget is zero
        if (!e && prm.repair) {
            bool zero = false;
            for (int s = lane; s < S; s += 32) zero |= b_fin[s] == 0;
            if (__any_sync(0xffffffffu, zero)) {
                uint32_t r = 0;
                if (lane == 0) r = repair_dev(b_fin, b_caps, S);
                e |= __shfl_sync(0xffffffffu, r, 0);
                __syncwarp();
            }
        }
        // on any error every budget is zero: the layout and gather after this kernel then copy
        // the window rows only and never index kept positions that were not written
        bool act = false;
        for (int s = lane; s < S; s += 32) {
            if (e) b_fin[s] = 0;
            const int64_t b = int64_t(b_fin[s]), n = int64_t(b_caps[s]);
            seg_active[s] = 0;
            if (e) {
                seg_mode[s] = MODE_NONE;
            } else if (prm.streaming) {
                seg_mode[s] = MODE_STREAM;
                seg_sink[s] = prm.sink < b ? prm.sink : b;
                seg_recent[s] = b - seg_sink[s];
            } else if (b == 0) {
                seg_mode[s] = MODE_NONE;
            } else if (b == n) {
                seg_mode[s] = MODE_ALL;
            } else if (adaptive && g_k > 0 && g_k <= N && b_fin[s] == b_raw[s]) {
                // per-segment top-b == the layer-wide selection restricted to s
                seg_mode[s] = MODE_THRESH;
                seg_T[s] = g_T;
            } else {
                seg_mode[s] = MODE_THRESH;
                seg_active[s] = 1;
                seg_prefix[s] = common;
                seg_krem[s] = b;
                act = true;
            }
        }
        act = __any_sync(0xffffffffu, act);
        if (lane == 0) {
            any_active = act ? 1 : 0;
            s_err = e;
            if (e && rank == 0) atomicOr(prm.err, e);
        }
    }
    __syncthreads();
    if (rank == 0) {
        for (int s = tid; s < S; s += kSelThreads) {
            prm.budgets[p * S + s] = int32_t(b_fin[s]);
            if (adaptive && prm.raw_counts) prm.raw_counts[p * S + s] = int32_t(b_raw[s]);
        }
    }

    stamp();
    // ---------------- Phase D: per-segment top-b (topk_decision, policies.hpp:80-93)
    if (any_active) {
        for (int pass = 0; pass < npass; ++pass) {
            if (pass == 0 && have_hist0) {
                for (int i = tid; i < S * 256; i += kSelThreads) agg[i] = hist0[i];
                __syncthreads();
            } else {
                radix_pass(pass);
            }
            for (int s = warp; s < S; s += kWarps) {
                if (!seg_active[s]) continue;
                const BinPick bp = find_bin(agg + s * 256, seg_krem[s], lane);
                if (lane == 0) {
                    seg_krem[s] -= bp.cum_above;
                    seg_prefix[s] |= KT(bp.bin) << lo_bit(pass);
                }
            }
            __syncthreads();
        }
        for (int s = tid; s < S; s += kSelThreads)
            if (seg_active[s]) {
                seg_T[s] = seg_prefix[s];
                seg_need[s] = seg_krem[s];
            }
    }
    __syncthreads();

    stamp();
    // ---------------- Phase E: keep mask and kept positions in flat order
    const int64_t wlo = lo + (hi - lo) * warp / kWarps, whi = lo + (hi - lo) * (warp + 1) / kWarps;
    const unsigned lt = (1u << lane) - 1u;
    for (int i = tid; i < kWarps * S * 2; i += kSelThreads) wcnt[i] = 0;
    __syncthreads();
    for (int s = 0; s < S; ++s) {
        const int64_t a = max(wlo, prm.off[s]), b = min(whi, prm.off[s + 1]);
        if (a >= b) continue;
        const int mode = seg_mode[s];
        uint32_t gt = 0, eq = 0;
        if (mode == MODE_THRESH) {
            const KT T = seg_T[s];
            // kEChunks chunks' loads in flight before any compare; per-lane counts, one warp sum
            for (int64_t base = a; base < b; base += 32 * kEChunks) {
                KT u[kEChunks];
#pragma unroll
                for (int c = 0; c < kEChunks; ++c) {
                    const int64_t e = base + c * 32 + lane;
                    u[c] = e < b ? key_at(e) : KT(0);
                }
#pragma unroll
                for (int c = 0; c < kEChunks; ++c) {
                    const bool ok = base + c * 32 + lane < b;
                    gt += (ok && u[c] > T) ? 1u : 0u;
                    eq += (ok && u[c] == T) ? 1u : 0u;
                }
            }
            gt = __reduce_add_sync(0xffffffffu, gt);
            eq = __reduce_add_sync(0xffffffffu, eq);
        } else if (mode == MODE_ALL) {
            gt = uint32_t(b - a);
        } else if (mode == MODE_STREAM) {
            const int64_t n = prm.off[s + 1] - prm.off[s];
            const int64_t pa = a - prm.off[s], pb = b - prm.off[s];
            const int64_t s_hi = seg_sink[s], r_lo = n - seg_recent[s];
            const int64_t c1 = max(int64_t(0), min(pb, s_hi) - pa);
            const int64_t c2 = max(int64_t(0), pb - max(pa, r_lo));
            gt = uint32_t(c1 + c2);
        }
        if (lane == 0) {
            wcnt[(warp * S + s) * 2 + 0] = gt;
            wcnt[(warp * S + s) * 2 + 1] = eq;
        }
    }
    __syncthreads();
    for (int s = tid; s < S; s += kSelThreads) {
        uint32_t gt = 0, eq = 0;
        for (int w = 0; w < kWarps; ++w) {
            gt += wcnt[(w * S + s) * 2 + 0];
            eq += wcnt[(w * S + s) * 2 + 1];
        }
        ccnt[s][0] = gt;
        ccnt[s][1] = eq;
    }
    stamp();
    cluster.sync();
    stamp();
    // cross-CTA prefix: T-equal elements and kept elements before this CTA
    __shared__ int64_t cta_kept_before;
    __shared__ int64_t seg_kept_before[kMaxSeg];
    for (int s = tid; s < S; s += kSelThreads) {
        int64_t eqb = 0, kept = 0;
        const int64_t need = seg_mode[s] == MODE_THRESH ? seg_need[s] : 0;
        for (unsigned rb = 0; rb < rank; rb += 8) {
            uint32_t rg[8], rq[8];  // eight lower ranks' counts per round, their remote loads in flight at once
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                rg[r] = rq[r] = 0u;
                if (rb + unsigned(r) < rank) {
                    const uint32_t* rc = cluster.map_shared_rank(&ccnt[0][0], rb + r);
                    rg[r] = rc[s * 2 + 0];
                    rq[r] = rc[s * 2 + 1];
                }
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int64_t g = rg[r], q = rq[r];
                const int64_t t = need - eqb;
                kept += g + (t <= 0 ? 0 : (t < q ? t : q));
                eqb += q;
            }
        }
        seg_eqb[s] = eqb;
        seg_kept_before[s] = kept;
    }
    __syncthreads();
    if (tid == 0) {
        int64_t t = 0;
        for (int s = 0; s < S; ++s) t += seg_kept_before[s];
        cta_kept_before = t;
    }
    // per segment, one warp: lane w takes warp w's counts; the T-equal counts of the warps
    // before it are an exclusive prefix sum over the lanes (kWarps == 32)
    static_assert(kWarps == 32, "lane per warp");
    for (int s = warp; s < S; s += kWarps) {
        const int64_t need = seg_mode[s] == MODE_THRESH ? seg_need[s] : 0;
        const int64_t g = wcnt[(lane * S + s) * 2 + 0], q = wcnt[(lane * S + s) * 2 + 1];
        int64_t inc = q;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        const int64_t eqb = seg_eqb[s] + inc - q;
        const int64_t t = need - eqb;
        wkept[lane * S + s] = g + (t <= 0 ? 0 : (t < q ? t : q));
        weqb[lane * S + s] = eqb;
    }
    __syncthreads();
    // kept elements before each warp: lane w's total over segments, exclusive prefix over lanes
    if (warp == 0) {
        int64_t tot = 0;
        for (int s = 0; s < S; ++s) tot += wkept[lane * S + s];
        int64_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        wkept_before[lane] = cta_kept_before + inc - tot;
    }
    __syncthreads();
    {
        int64_t run_kept = wkept_before[warp];
        uint8_t* keep_out = prm.keep ? prm.keep + p * N : nullptr;
        int32_t* kp = prm.kept_pos ? prm.kept_pos + p * prm.kept_stride : nullptr;
        for (int s = 0; s < S; ++s) {
            // everything the element loop reads is loaded once here: its byte stores may alias
            // any generic address, which would otherwise force a reload per element
            const int64_t off_s = prm.off[s], off_e = prm.off[s + 1];
            const int64_t a = max(wlo, off_s), b = min(whi, off_e);
            if (a >= b) continue;
            const int mode = seg_mode[s];
            const KT T = seg_T[s];
            const int64_t need = seg_need[s];
            const int64_t n = off_e - off_s;
            const int64_t sink = seg_sink[s], recent_lo = n - seg_recent[s];
            int64_t run_eq = weqb[warp * S + s];
            // 32-bit element offsets from the warp's range start (ranges fit 32 bits)
            const int len = int(b - a);
            const int pos0 = int(a - off_s);
            auto emit = [&](int j, bool valid, bool keep) {
                const unsigned bk = __ballot_sync(0xffffffffu, keep);
                ADAKV_DCHECK(!(keep && kp) || run_kept + __popc(bk & lt) < prm.kept_stride);
                if (keep && kp) kp[run_kept + __popc(bk & lt)] = int32_t(pos0 + j);
                if (valid && keep_out) keep_out[a + j] = keep ? 1 : 0;
                run_kept += __popc(bk);
            };
            if (mode == MODE_THRESH) {
                // kEChunks chunks' key loads issued ahead of the stores (which may alias them)
                for (int o = 0; o < len; o += 32 * kEChunks) {
                    KT u[kEChunks];
#pragma unroll
                    for (int c = 0; c < kEChunks; ++c) {
                        const int j = o + c * 32 + lane;
                        u[c] = j < len ? key_at(a + j) : KT(0);
                    }
#pragma unroll
                    for (int c = 0; c < kEChunks; ++c) {
                        if (o + c * 32 >= len) break;  // warp-uniform
                        const int j = o + c * 32 + lane;
                        const bool valid = j < len;
                        const bool is_eq = valid && u[c] == T;
                        const unsigned beq = __ballot_sync(0xffffffffu, is_eq);
                        const int64_t eqr = run_eq + __popc(beq & lt);
                        emit(j, valid, valid && (u[c] > T || (is_eq && eqr < need)));
                        run_eq += __popc(beq);
                    }
                }
            } else {
                for (int o = 0; o < len; o += 32) {
                    const int j = o + lane;
                    const bool valid = j < len;
                    const int pos = pos0 + j;
                    bool keep = false;
                    if (mode == MODE_ALL) keep = valid;
                    else if (mode == MODE_STREAM) keep = valid && (pos < sink || pos >= recent_lo);
                    emit(j, valid, keep);
                }
            }
        }
    }
    stamp();
    cluster.sync();  // keep peer shared memory alive until every CTA is done reading it
    stamp();
}

}  // namespace

size_t select_smem_bytes(int S) {
    return size_t(4) * (2 * S * 256 + S * 256 + S * 256 + kWarps * S * 2) + size_t(8) * 2 * kWarps * S +
           size_t(4) * kWarps * 256;
}
// the same without the second histogram buffer and the kept first-digit histograms (lean)
size_t select_smem_bytes_lean(int S) {
    return select_smem_bytes(S) - size_t(4) * 2 * S * 256;
}
constexpr size_t kSelSmemCap = 220 * 1024;  // dynamic shared memory budget per CTA

// The kernels' attributes are set once per device, to the most dynamic shared memory the
// device allows beside their static shared memory (and non-portable cluster sizes), so no
// launch ever changes them (concurrent launches of different sizes cannot race).
using SelKernel = void (*)(const SelParams, unsigned long long*);
static SelKernel select_fn(bool key64, bool nonneg) {
    return key64 ? (nonneg ? select_kernel<double, true> : select_kernel<double, false>)
                 : (nonneg ? select_kernel<float, true> : select_kernel<float, false>);
}

static cudaError_t select_prepare(SelKernel fn, size_t* max_dyn) {
    static std::mutex mu;
    static std::map<std::pair<int, SelKernel>, size_t> cap;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cap.find({dev, fn});
    if (it != cap.end()) {
        *max_dyn = it->second;
        return cudaSuccess;
    }
    cudaFuncAttributes fa{};
    int optin = 0;
    e = cudaFuncGetAttributes(&fa, fn);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t c = std::min(kSelSmemCap, size_t(optin) - fa.sharedSizeBytes);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c));
    if (e == cudaSuccess) cap[{dev, fn}] = c;
    *max_dyn = c;
    return e;
}

// dynamic shared memory of a select launch with CS CTAs per cluster; sets cache_keys
static size_t select_launch_smem(bool key64, const SelParams& prm, int CS, size_t max_dyn, int* cache_keys) {
    size_t smem = prm.lean ? select_smem_bytes_lean(prm.S) : select_smem_bytes(prm.S);
    const size_t key_bytes = size_t(ceil_div(prm.N, CS)) * (key64 ? 8 : 4) + 16;  // + vector-read slack
    *cache_keys = smem + key_bytes <= max_dyn;
    return *cache_keys ? smem + key_bytes : smem;
}

// clusters of CS CTAs (smem bytes each) the device holds at once
static int select_fit(SelKernel fn, int CS, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, SelKernel, int, size_t>, int> memo;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, fn, CS, smem);
    std::lock_guard<std::mutex> lock(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    int n = 0;
    size_t max_dyn = 0;
    if (select_prepare(fn, &max_dyn) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(CS));
        cfg.blockDim = dim3(kSelThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = unsigned(CS);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) n = 0;
    }
    cudaGetLastError();
    memo[key] = n;
    return n;
}

adakv_status launch_select(bool key64, int64_t P, const SelParams& prm, cudaStream_t stream) {
    if (P == 0) return ADAKV_OK;
    // Cluster size: the largest (<= 16, and no more than ~16K keys per CTA) for which every
    // problem of the call is resident at once -- one wave; a problem's latency is mostly its
    // per-pass barriers, so one wave of smaller clusters beats two of larger ones (config 2,
    // 32 problems of 262K keys: 4 CTAs streaming their slices from L2, 124 us, against 8 CTAs
    // with the keys in shared memory in two waves, 207 us).  No size fits one wave: up to 8.
    const int64_t per_cta = 16384;
    const int64_t want = ceil_div(prm.N, per_cta);
    int CS = int(want < 1 ? 1 : (want > 8 ? 8 : want));
    const SelKernel fn = select_fn(key64, prm.nonneg != 0);
    size_t max_dyn = 0;
    ADAKV_CUDA_TRY(select_prepare(fn, &max_dyn));
    // per-segment histograms (~4.75 KB per segment) beside the per-warp ones fit up to 39
    // segments (KV groups) per problem on B200; more take the lean layout (~2.75 KB per
    // segment, up to 68: one histogram buffer and an extra cluster barrier per pass)
    SelParams lp = prm;
    lp.lean = select_smem_bytes(prm.S) > max_dyn ? 1 : 0;
    if (select_smem_bytes_lean(prm.S) > max_dyn)
        return fail(ADAKV_UNSUPPORTED, "selection: too many segments (KV groups) per problem for shared memory");
    int cache_keys = 0;
    for (int c = int(want < 1 ? 1 : (want < kMaxSelCS ? want : kMaxSelCS)); c >= 1; --c) {
        if (select_fit(fn, c, select_launch_smem(key64, lp, c, max_dyn, &cache_keys)) >= P) {
            CS = c;
            break;
        }
    }
    if (const char* e = std::getenv("ADAKV_SELECT_CS")) CS = std::max(1, std::min(kMaxSelCS, std::atoi(e)));
    const size_t smem = select_launch_smem(key64, lp, CS, max_dyn, &cache_keys);
    lp.cache_keys = cache_keys;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(P * CS));
    cfg.blockDim = dim3(kSelThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(CS);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ADAKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, lp, g_sel_dbg));
    return ADAKV_OK;
}

extern "C" void adakv_debug_set_select_timestamps(void* buf) { g_sel_dbg = static_cast<unsigned long long*>(buf); }

// ---------------------------------------------------------------- standalone budget kernels
__global__ void budget_kernel(int op, const double* quotas_in, const int64_t* a_in, int64_t h,
                              int64_t total, double alpha, double bmax, double bmin,
                              const int64_t* caps_in, int64_t* out, double* quotas,
                              uint64_t* caps, uint64_t* tmp_a, uint64_t* tmp_o, uint32_t* err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int64_t i = 0; i < h; ++i) caps[i] = caps_in ? uint64_t(caps_in[i]) : kAmpleCap;
    uint32_t e = 0;
    switch (op) {
        case 0:  // apportion
            for (int64_t i = 0; i < h; ++i) quotas[i] = quotas_in[i];
            e = apportion_dev(quotas, int(h), uint64_t(total), caps, tmp_o);
            break;
        case 1:  // uniform
            e = uniform_dev(uint64_t(total), int(h), caps, quotas, tmp_o);
            break;
        case 2:  // safeguard
            for (int64_t i = 0; i < h; ++i) tmp_a[i] = uint64_t(a_in[i]);
            e = safeguard_dev(tmp_a, uint64_t(total), int(h), alpha, caps, quotas, tmp_o);
            break;
        case 3:  // repair (in place)
            for (int64_t i = 0; i < h; ++i) tmp_o[i] = uint64_t(a_in[i]);
            e = repair_dev(tmp_o, caps, int(h));
            break;
        case 4:  // pyramid
            e = pyramid_dev(uint64_t(total), int(h), bmax, bmin, quotas, caps, tmp_o);
            break;
    }
    *err = e;
    for (int64_t i = 0; i < h; ++i) out[i] = int64_t(tmp_o[i]);
}

}  // namespace adakv_b200
