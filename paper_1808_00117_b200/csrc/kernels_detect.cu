// kernels_detect.cu -- A1 "detect": which pages changed
// since the last commit.  Reading Q1: the paper's write-fault
// MarkPageAsDirty (Alg. 1) becomes a content test, because
// GPU stores cannot be trapped:
//   COMPARE: any byte of page i differs from the device mirror  (HBM: 2 reads)
//   HASH   : XXH3-64 of the zero-padded slot differs from table  (HBM: 1 read)
//
// Both kernels are persistent grid-stride loops sized to the SM count.
//  * compare: one warp per 4 KiB segment; 256-bit (LDG.256) streaming loads,
//    4 per lane per operand = 8 x 32 B in flight per lane; warp vote.
//  * hash: one warp per page (two 4 KiB pages per warp), lane = 4*b + p owns
//    block b (1 KiB) and u64 lanes {2p, 2p+1} of every stripe, so the
//    per-block "accumulate" sums stay in registers (no shuffles); the serial
//    scramble chain across blocks runs on 4 lanes per page fed by 8 shuffles
//    per 8 KiB.  XXH3 structure: xxhash 0.8 long-input loop (see
//    DESIGN.md "XXH3 on the GPU"), written here independently of oracle/.
#include <algorithm>

#include "crum_internal.cuh"

namespace crum {

// ---------------------------------------------------------------------------
// Streaming vector loads (read-only path, no L1 allocation).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ld256(const void *p, uint32_t (&r)[8]) {
    asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p));
}
__device__ __forceinline__ uint4 ld128(const void *p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

// ---------------------------------------------------------------------------
// COMPARE detect.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_detect_compare(
    const DevRegion *__restrict__ regs, const uint32_t *__restrict__ cmp_idx,
    const uint64_t *__restrict__ cmp_seg, uint32_t n_cmp, uint64_t s_lo, uint64_t s_hi,
    const uint8_t *__restrict__ force, uint8_t *__restrict__ flags, uint8_t tag) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    uint64_t r_lo = 1, r_hi = 0;  // cached segment range of the current region
    DevRegion R{};
    for (uint64_t s = s_lo + (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5); s < s_hi; s += nwarps) {
        if (s < r_lo || s >= r_hi) {
            uint32_t r = upper_region(cmp_seg, n_cmp, s);
            R = regs[__ldg(cmp_idx + r)];
            r_lo = __ldg(cmp_seg + r);
            r_hi = __ldg(cmp_seg + r + 1);
        }
        const uint64_t si = s - r_lo;
        const uint64_t off = si << kSegLog2;
        const uint64_t g = R.page_base + (si >> (R.log2p - kSegLog2));
        if (__ldg(force + g)) continue;  // already dirty: no need to read the bytes
        const uint64_t len = R.bytes - off;
        const uint8_t *a = R.base + off;
        const uint8_t *b = R.mirror + off;
        uint32_t x = 0;
        if (len >= kSegBytes) {
            if (R.aligned32) {
                uint32_t va[4][8], vb[4][8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    ld256(a + i * 1024 + lane * 32, va[i]);
                    ld256(b + i * 1024 + lane * 32, vb[i]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) x |= va[i][j] ^ vb[i][j];
            } else {
                uint4 va[8], vb[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    va[i] = ld128(a + i * 512 + lane * 16);
                    vb[i] = ld128(b + i * 512 + lane * 16);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    x |= (va[i].x ^ vb[i].x) | (va[i].y ^ vb[i].y) | (va[i].z ^ vb[i].z) |
                         (va[i].w ^ vb[i].w);
            }
        } else {  // logical tail of a partial last page (reading Q7): bytewise
            for (uint32_t o = lane; o < len; o += 32) x |= (uint32_t)(a[o] ^ b[o]);
        }
        if (__any_sync(0xffffffffu, x != 0) && lane == 0) flags[g] = tag;
    }
}

// ---------------------------------------------------------------------------
// XXH3-64 (seed 0, default 192-byte secret), long-input path, per page slot.
// ---------------------------------------------------------------------------
constexpr uint8_t kSecretBytes[192] = {
    0xb8, 0xfe, 0x6c, 0x39, 0x23, 0xa4, 0x4b, 0xbe, 0x7c, 0x01, 0x81, 0x2c, 0xf7, 0x21, 0xad, 0x1c,
    0xde, 0xd4, 0x6d, 0xe9, 0x83, 0x90, 0x97, 0xdb, 0x72, 0x40, 0xa4, 0xa4, 0xb7, 0xb3, 0x67, 0x1f,
    0xcb, 0x79, 0xe6, 0x4e, 0xcc, 0xc0, 0xe5, 0x78, 0x82, 0x5a, 0xd0, 0x7d, 0xcc, 0xff, 0x72, 0x21,
    0xb8, 0x08, 0x46, 0x74, 0xf7, 0x43, 0x24, 0x8e, 0xe0, 0x35, 0x90, 0xe6, 0x81, 0x3a, 0x26, 0x4c,
    0x3c, 0x28, 0x52, 0xbb, 0x91, 0xc3, 0x00, 0xcb, 0x88, 0xd0, 0x65, 0x8b, 0x1b, 0x53, 0x2e, 0xa3,
    0x71, 0x64, 0x48, 0x97, 0xa2, 0x0d, 0xf9, 0x4e, 0x38, 0x19, 0xef, 0x46, 0xa9, 0xde, 0xac, 0xd8,
    0xa8, 0xfa, 0x76, 0x3f, 0xe3, 0x9c, 0x34, 0x3f, 0xf9, 0xdc, 0xbb, 0xc7, 0xc7, 0x0b, 0x4f, 0x1d,
    0x8a, 0x51, 0xe0, 0x4b, 0xcd, 0xb4, 0x59, 0x31, 0xc8, 0x9f, 0x7e, 0xc9, 0xd9, 0x78, 0x73, 0x64,
    0xea, 0xc5, 0xac, 0x83, 0x34, 0xd3, 0xeb, 0xc3, 0xc5, 0x81, 0xa0, 0xff, 0xfa, 0x13, 0x63, 0xeb,
    0x17, 0x0d, 0xdd, 0x51, 0xb7, 0xf0, 0xda, 0x49, 0xd3, 0x16, 0x55, 0x26, 0x29, 0xd4, 0x68, 0x9e,
    0x2b, 0x16, 0xbe, 0x58, 0x7d, 0x47, 0xa1, 0xfc, 0x8f, 0xf8, 0xb8, 0xd1, 0x7a, 0xd0, 0x31, 0xce,
    0x45, 0xcb, 0x3a, 0x8f, 0x95, 0x16, 0x04, 0x28, 0xaf, 0xd7, 0xfb, 0xca, 0xbb, 0x4b, 0x40, 0x7e,
};

struct XxhConsts {
    uint64_t w[24];      // secret as 24 aligned little-endian words (stripe keys, scramble keys 16..23)
    uint64_t last[8];    // words at byte offset 121 + 8l (the last stripe)
    uint64_t merge[8];   // words at byte offset 11 + 8l (merge)
    uint64_t init[8];    // initial accumulators
};

constexpr uint64_t le64_at(int off) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | kSecretBytes[off + i];
    return v;
}

constexpr XxhConsts make_consts() {
    XxhConsts c{};
    for (int i = 0; i < 24; ++i) c.w[i] = le64_at(8 * i);
    for (int l = 0; l < 8; ++l) c.last[l] = le64_at(121 + 8 * l);
    for (int l = 0; l < 8; ++l) c.merge[l] = le64_at(11 + 8 * l);
    c.init[0] = 0xC2B2AE3Dull;            // PRIME32_3
    c.init[1] = 0x9E3779B185EBCA87ull;    // PRIME64_1
    c.init[2] = 0xC2B2AE3D27D4EB4Full;    // PRIME64_2
    c.init[3] = 0x165667B19E3779F9ull;    // PRIME64_3
    c.init[4] = 0x85EBCA77C2B2AE63ull;    // PRIME64_4
    c.init[5] = 0x85EBCA77ull;            // PRIME32_2
    c.init[6] = 0x27D4EB2F165667C5ull;    // PRIME64_5
    c.init[7] = 0x9E3779B1ull;            // PRIME32_1
    return c;
}

__constant__ XxhConsts c_xxh = make_consts();

constexpr uint64_t kP32_1 = 0x9E3779B1ull;
constexpr uint64_t kP64_1 = 0x9E3779B185EBCA87ull;
constexpr uint64_t kMx1 = 0x165667919E3779F9ull;

// Per-lane constants: lane p (= lane & 3) owns accumulator lanes 2p, 2p+1.
struct LaneKeys {
    const uint64_t *sw;        // stripe keys in shared memory: sw[s] = word (s + 2p), s = 0..16
    uint64_t last0, last1;     // last-stripe keys for lanes 2p, 2p+1
    uint64_t scr0, scr1;       // scramble keys
    uint64_t mrg0, mrg1;       // merge keys
    uint64_t init0, init1;     // initial accumulators
};

// The 24 secret words are staged in shared memory (keeps ~34 registers per
// thread free for loads in flight); call with all threads, then sync.
__device__ __forceinline__ void stage_secret(uint64_t *s_w) {
    if (threadIdx.x < 24) s_w[threadIdx.x] = c_xxh.w[threadIdx.x];
}

__device__ __forceinline__ void load_lane_keys(LaneKeys &k, uint32_t p, const uint64_t *s_w) {
    k.sw = s_w + 2 * p;
    k.last0 = c_xxh.last[2 * p];
    k.last1 = c_xxh.last[2 * p + 1];
    k.scr0 = c_xxh.w[16 + 2 * p];
    k.scr1 = c_xxh.w[17 + 2 * p];
    k.mrg0 = c_xxh.merge[2 * p];
    k.mrg1 = c_xxh.merge[2 * p + 1];
    k.init0 = c_xxh.init[2 * p];
    k.init1 = c_xxh.init[2 * p + 1];
}

// One stripe's contribution to accumulator lanes (2p, 2p+1):
//   acc[l]   += lo32(v_l ^ key_l) * hi32(v_l ^ key_l)
//   acc[l^1] += v_l
__device__ __forceinline__ void accum16(uint64_t &a0, uint64_t &a1, uint4 d, uint64_t s0,
                                        uint64_t s1) {
    const uint64_t v0 = ((uint64_t)d.y << 32) | d.x;
    const uint64_t v1 = ((uint64_t)d.w << 32) | d.z;
    const uint64_t k0 = v0 ^ s0, k1 = v1 ^ s1;
    a0 += (uint64_t)(uint32_t)k0 * (uint32_t)(k0 >> 32) + v1;
    a1 += (uint64_t)(uint32_t)k1 * (uint32_t)(k1 >> 32) + v0;
}

__device__ __forceinline__ uint64_t scramble(uint64_t a, uint64_t key) {
    a ^= a >> 47;
    a ^= key;
    return a * kP32_1;
}

// 16 bytes of a page slot at byte offset `off`; bytes at or beyond `len` read
// as zero (zero-padded slot, reading Q7).
__device__ __forceinline__ uint4 ld_slot16(const uint8_t *pg, uint64_t off, uint64_t len) {
    if (off + 16 <= len) return ld128(pg + off);
    uint32_t w[4] = {0, 0, 0, 0};
    for (uint32_t i = 0; i < 16; ++i)
        if (off + i < len) w[i >> 2] |= (uint32_t)pg[off + i] << (8 * (i & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// XXH3-64 of this lane's page slot.  G = blocks per page per 8 KiB step
// (8 for P >= 8 KiB; 4 for P = 4 KiB, two pages per warp).  `pg` is the page
// base of the lane's group, `len` its logical length (<= P), bpp = P / 1024.
// Result is valid on the group's chain lanes (lane % (4G) < 4).
template <int G, bool TAIL>
__device__ __forceinline__ uint64_t xxh3_slot(const uint8_t *__restrict__ pg, uint64_t len,
                                              uint32_t bpp, uint32_t lane, const LaneKeys &k) {
    const uint32_t p = lane & 3;
    const uint32_t bl = (lane >> 2) % G;       // block slot within the group
    const bool chain = (lane % (4 * G)) < 4;
    uint64_t c0 = k.init0, c1 = k.init1;
    const uint32_t steps = bpp / G;
    for (uint32_t t = 0; t < steps; ++t) {
        const uint32_t bi = t * G + bl;        // block index within the page
        const uint64_t boff = (uint64_t)bi * 1024 + p * 16;
        uint4 d[16];
#pragma unroll
        for (int s = 0; s < 16; ++s)
            d[s] = TAIL ? ld_slot16(pg, boff + s * 64, len) : ld128(pg + boff + s * 64);
        uint64_t a0 = 0, a1 = 0;
#pragma unroll
        for (int s = 0; s < 15; ++s) accum16(a0, a1, d[s], k.sw[s], k.sw[s + 1]);
        const bool lastblk = (bi == bpp - 1);
        accum16(a0, a1, d[15], lastblk ? k.last0 : k.sw[15], lastblk ? k.last1 : k.sw[16]);
        // serial chain over the step's G blocks (chain lanes only keep results)
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const uint64_t x0 = __shfl_sync(0xffffffffu, a0, lane + 4 * j);
            const uint64_t x1 = __shfl_sync(0xffffffffu, a1, lane + 4 * j);
            c0 += x0;
            c1 += x1;
            if (t * G + j != bpp - 1) {
                c0 = scramble(c0, k.scr0);
                c1 = scramble(c1, k.scr1);
            }
        }
    }
    // merge: r = P * PRIME64_1 + sum_i fold64((acc[2i]^m[2i]) * (acc[2i+1]^m[2i+1]))
    const uint64_t x = c0 ^ k.mrg0, y = c1 ^ k.mrg1;
    uint64_t m = (x * y) ^ __umul64hi(x, y);
    m += __shfl_xor_sync(0xffffffffu, m, 1);
    m += __shfl_xor_sync(0xffffffffu, m, 2);
    uint64_t r = (uint64_t)bpp * 1024 * kP64_1 + m;
    r ^= r >> 37;
    r *= kMx1;
    r ^= r >> 32;
    (void)chain;
    return r;
}

// ---------------------------------------------------------------------------
// HASH detect: warp per page group (1 page, or 2 pages when P = 4 KiB).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 2) k_detect_hash(
    const DevRegion *__restrict__ regs, const uint32_t *__restrict__ hash_idx,
    const uint64_t *__restrict__ hash_grp, uint32_t n_hash, uint64_t w_lo, uint64_t w_hi,
    uint8_t *__restrict__ flags, uint64_t *__restrict__ newhash, uint8_t tag) {
    const uint32_t lane = threadIdx.x & 31;
    __shared__ uint64_t s_w[24];
    stage_secret(s_w);
    __syncthreads();
    LaneKeys k;
    load_lane_keys(k, lane & 3, s_w);
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    uint64_t r_lo = 1, r_hi = 0;
    DevRegion R{};
    for (uint64_t w = w_lo + (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5); w < w_hi; w += nwarps) {
        if (w < r_lo || w >= r_hi) {
            uint32_t r = upper_region(hash_grp, n_hash, w);
            R = regs[__ldg(hash_idx + r)];
            r_lo = __ldg(hash_grp + r);
            r_hi = __ldg(hash_grp + r + 1);
        }
        const uint64_t P = 1ull << R.log2p;
        const uint32_t bpp = (uint32_t)(P >> 10);
        uint64_t h;
        uint64_t page;
        bool valid;
        if (R.log2p == 12) {  // two 4 KiB pages per warp
            page = (w - r_lo) * 2 + (lane >> 4);
            valid = page < R.n_pages;
            const uint64_t pg = valid ? page : page - 1;  // idle half recomputes its neighbour
            const uint64_t len = min(P, R.bytes - (pg << 12));
            const uint8_t *base = R.base + (pg << 12);
            const bool tail = __any_sync(0xffffffffu, len < P);
            h = tail ? xxh3_slot<4, true>(base, len, bpp, lane, k)
                     : xxh3_slot<4, false>(base, len, bpp, lane, k);
        } else {
            page = w - r_lo;
            valid = true;
            const uint64_t len = min(P, R.bytes - (page << R.log2p));
            const uint8_t *base = R.base + (page << R.log2p);
            h = (len < P) ? xxh3_slot<8, true>(base, len, bpp, lane, k)
                          : xxh3_slot<8, false>(base, len, bpp, lane, k);
        }
        const uint32_t G = (R.log2p == 12) ? 4 : 8;
        if (valid && (lane % (4 * G)) == 0) {
            const uint64_t g = R.page_base + page;
            const uint64_t old = R.table[page];
            newhash[g] = h;
            flags[g] = (h != old) ? tag : 0;
        }
    }
}

// Named barriers (bar.sync / bar.arrive) pair the compute and chain warps of
// the TMA-fed hash kernels below.
__device__ __forceinline__ void bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------------------
// HASH detect for large pages, TMA-fed (the default for P >= 64 KiB): three
// persistent CTAs per SM (three independent scramble chains -- a page's chain
// is serial, so chains per SM bound the rate).  Warp 5 (the "loader")
// streams each 32 KiB round of the CTA's pages into a 2-stage shared-memory
// ring with one cp.async.bulk (UBLKCP) per round, completing on the stage's
// FULL mbarrier (tx bytes); the partial rounds of a region's last page are
// copied by the loader's lanes with zero fill instead.  Warps 0..3 compute
// the 32 block accumulate sums of a round from shared memory (same lane
// layout as above) and release the stage on its EMPTY mbarrier (4
// arrivals); warp 4 runs the scramble chain over the block sums (named
// barriers 1-4, 160 threads).  192 KiB per SM are in flight with no
// registers held.
// ---------------------------------------------------------------------------
constexpr int kTmaCompute = 4;                                  // compute warps
constexpr int kTmaRB = kTmaCompute * 8;                           // blocks per round
constexpr int kTmaStages = 2;                                    // default ring depth
constexpr uint32_t kTmaRound = (uint32_t)kTmaRB * 1024u;         // 32 KiB
constexpr int kTmaChainThreads = (kTmaCompute + 1) * 32;          // named-barrier participants
constexpr int kTmaThreads = kTmaChainThreads + 32;                // + loader warp
constexpr int kTmaCtasPerSm = 3;                                  // 3 scramble chains per SM

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kTmaThreads, kTmaCtasPerSm) k_detect_hash_tma(
    const DevRegion *__restrict__ regs, const uint32_t *__restrict__ big_idx,
    const uint64_t *__restrict__ big_pg, uint32_t n_big, uint64_t w_lo, uint64_t w_hi,
    uint8_t *__restrict__ flags, uint64_t *__restrict__ newhash, uint8_t tag, uint32_t nst) {
    extern __shared__ __align__(1024) uint8_t ring[];  // nst x kTmaRound
    __shared__ uint64_t S[2][kTmaRB][8];
    __shared__ __align__(8) uint64_t full_bar[kTmaStages], empty_bar[kTmaStages];
    __shared__ uint64_t sw[24], slast[8], smerge[8], sinit[8];
    if (threadIdx.x < 24) sw[threadIdx.x] = c_xxh.w[threadIdx.x];
    if (threadIdx.x < 8) {
        slast[threadIdx.x] = c_xxh.last[threadIdx.x];
        smerge[threadIdx.x] = c_xxh.merge[threadIdx.x];
        sinit[threadIdx.x] = c_xxh.init[threadIdx.x];
    }
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < nst; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], kTmaCompute);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t q = 0;  // round counter across this CTA's pages (stage = q % nst, use = q / nst)
    uint64_t r_lo = 1, r_hi = 0;
    DevRegion R{};
    for (uint64_t w = w_lo + blockIdx.x; w < w_hi; w += gridDim.x) {
        if (w < r_lo || w >= r_hi) {
            const uint32_t r = upper_region(big_pg, n_big, w);
            R = regs[__ldg(big_idx + r)];
            r_lo = __ldg(big_pg + r);
            r_hi = __ldg(big_pg + r + 1);
        }
        const uint64_t page = w - r_lo;
        const uint64_t P = 1ull << R.log2p;
        const uint32_t bpp = (uint32_t)(P >> 10);
        const uint32_t rounds = bpp / kTmaRB;
        const uint64_t len = min(P, R.bytes - (page << R.log2p));
        const uint8_t *pg = R.base + (page << R.log2p);
        if (warp == kTmaCompute + 1) {
            // loader
            for (uint32_t rr = 0; rr < rounds; ++rr, ++q) {
                const uint32_t st = q % nst, use = q / nst;
                if (use) mbar_wait(&empty_bar[st], (use - 1) & 1);
                uint8_t *dst = ring + (size_t)st * kTmaRound;
                const uint64_t off = (uint64_t)rr * kTmaRound;
                if (off + kTmaRound <= len) {
                    if (lane == 0) {
                        mbar_arrive_tx(&full_bar[st], kTmaRound);
                        bulk_g2s(dst, pg + off, kTmaRound, &full_bar[st]);
                    }
                } else {
                    // partial round of a region's last page: zero-padded copy
                    for (uint32_t o = lane * 16; o < kTmaRound; o += 512)
                        *reinterpret_cast<uint4 *>(dst + o) = ld_slot16(pg, off + o, len);
                    // order these generic-proxy stores before any later
                    // cp.async.bulk (async proxy) into the same stage
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full_bar[st]);
                }
            }
        } else if (warp < kTmaCompute) {
            const uint32_t p = lane & 3, b = lane >> 2;
            for (uint32_t rr = 0; rr < rounds; ++rr, ++q) {
                const uint32_t st = q % nst, use = q / nst;
                const uint32_t buf = q & 1;
                const uint32_t bl = warp * 8 + b;  // block within the round
                const uint32_t bi = rr * kTmaRB + bl;
                mbar_wait(&full_bar[st], use & 1);
                const uint8_t *src = ring + (size_t)st * kTmaRound + bl * 1024 + p * 16;
                uint4 d[16];
#pragma unroll
                for (int s2 = 0; s2 < 16; ++s2) d[s2] = *reinterpret_cast<const uint4 *>(src + s2 * 64);
                // Release the stage as soon as the loads have LANDED, not when
                // they are issued: the arrive is made data-dependent on every
                // loaded register (xor fold & a runtime zero the compiler cannot
                // see through), so its address waits on the LDS scoreboard.
                // An arrive right after the LDS issue let the next
                // cp.async.bulk overwrite the stage while reads were still in
                // flight (rare wrong hashes under load).
                uint32_t fold = 0;
#pragma unroll
                for (int s2 = 0; s2 < 16; ++s2) fold ^= d[s2].x ^ d[s2].y ^ d[s2].z ^ d[s2].w;
                const uint32_t dep = fold & (nst >> 16);  // nst <= kTmaStages: always 0
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[st] + dep);
                uint64_t a0 = 0, a1 = 0;
#pragma unroll
                for (int s2 = 0; s2 < 15; ++s2) accum16(a0, a1, d[s2], sw[s2 + 2 * p], sw[s2 + 2 * p + 1]);
                const bool lastblk = (bi == bpp - 1);
                accum16(a0, a1, d[15], lastblk ? slast[2 * p] : sw[15 + 2 * p],
                        lastblk ? slast[2 * p + 1] : sw[16 + 2 * p]);
                if (q >= 2) bar_sync(3 + buf, kTmaChainThreads);  // the chain has drained this buffer
                S[buf][bl][2 * p] = a0;
                S[buf][bl][2 * p + 1] = a1;
                bar_arrive(1 + buf, kTmaChainThreads);
            }
        } else {
            const uint32_t l = lane & 7;
            const uint64_t key = sw[16 + l];
            uint64_t acc = sinit[l];
            for (uint32_t rr = 0; rr < rounds; ++rr, ++q) {
                const uint32_t buf = q & 1;
                bar_sync(1 + buf, kTmaChainThreads);
                const uint32_t b0 = rr * kTmaRB;
#pragma unroll 8
                for (int j = 0; j < kTmaRB; ++j) {
                    acc += S[buf][j][l];
                    if (b0 + j != bpp - 1) acc = scramble(acc, key);
                }
                // arrive once the block sums have landed (acc depends on all of
                // them; nst >> 16 is a runtime zero), so the compute warps'
                // next stores to S[buf] cannot overtake a read still in flight
                bar_arrive(3 + buf + (uint32_t)(acc & (nst >> 16)), kTmaChainThreads);
            }
            const uint64_t x = acc ^ smerge[l];
            const uint64_t y = __shfl_down_sync(0xffffffffu, x, 1);
            uint64_t m = ((l & 1) == 0) ? ((x * y) ^ __umul64hi(x, y)) : 0;
            m += __shfl_xor_sync(0xffffffffu, m, 2);
            m += __shfl_xor_sync(0xffffffffu, m, 4);
            uint64_t h = P * kP64_1 + m;
            h ^= h >> 37;
            h *= kMx1;
            h ^= h >> 32;
            if (lane == 0) {
                const uint64_t g = R.page_base + page;
                newhash[g] = h;
                flags[g] = (h != R.table[page]) ? tag : 0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// HASH detect for large pages, TMA-fed, PAGE GROUPS (default for P >= 64 KiB).
// A page's scramble chain is serial (acc <- scramble(acc + S_b) per 1 KiB
// block) and uses 8 lanes; a CTA that hashes one page at a time leaves 24
// chain lanes idle and, measured, the chain warp competing for issue slots
// with the compute warps bounded short runs (0.82-0.87 of peak on C2; either
// half alone reached 0.99).  Here a CTA hashes TWO pages (big-page indices
// 2t and 2t+1 of the range) in lock step: every 32 KiB round carries 16
// blocks of each ("half" h = 0, 1), compute warps 2h and 2h+1 produce that
// half's block sums, and the chain warp runs both chains at once (lanes
// 8h..8h+7), so a round costs 16 serial chain steps instead of 32.  Pages of
// different sizes (a pair straddling regions) simply finish at different
// rounds; the idle half loads nothing.  Ring, release rule and named barriers
// as in k_detect_hash_tma.
// ---------------------------------------------------------------------------
constexpr int kPairStages = 2;

struct PairHalf {
    const uint8_t *pg;   // page base
    uint64_t len;        // logical bytes of the page (<= P)
    uint64_t g;          // global page id
    uint64_t old;        // stored hash (table entry)
    uint64_t P;
    uint32_t bpp;        // 1 KiB blocks per page
    uint32_t rounds;     // bpp / (32 / NP); 0 = no page in this slot
};

__device__ __forceinline__ void pair_half(const DevRegion *__restrict__ regs, const uint32_t *__restrict__ big_idx,
                                          const uint64_t *__restrict__ big_pg, uint32_t n_big, uint64_t w,
                                          uint64_t w_hi, uint32_t seg_blocks, PairHalf &h) {
    if (w >= w_hi) {
        h.rounds = 0;
        h.bpp = 0;
        return;
    }
    const uint32_t r = upper_region(big_pg, n_big, w);
    const DevRegion R = regs[__ldg(big_idx + r)];
    const uint64_t page = w - __ldg(big_pg + r);
    h.P = 1ull << R.log2p;
    h.bpp = (uint32_t)(h.P >> 10);
    h.rounds = h.bpp / seg_blocks;
    h.len = min(h.P, R.bytes - (page << R.log2p));
    h.pg = R.base + (page << R.log2p);
    h.g = R.page_base + page;
    h.old = R.table[page];
}

// NP = 2 pages hashed together: a 32 KiB round carries 16 blocks of each
// page; compute warp w serves page w / 2; chain lanes 8h..8h+7 run page h's
// chain.  (Four pages per CTA, 8 chain steps per round, measured slower:
// 0.865 vs 0.887 of peak on C2 64 KiB, 0.997 vs 1.021 on C4; removed.)
constexpr int NP = 2;
__global__ void __launch_bounds__(kTmaThreads, kTmaCtasPerSm) k_detect_hash_pair(
    const DevRegion *__restrict__ regs, const uint32_t *__restrict__ big_idx,
    const uint64_t *__restrict__ big_pg, uint32_t n_big, uint64_t w_lo, uint64_t w_hi,
    uint8_t *__restrict__ flags, uint64_t *__restrict__ newhash, uint8_t tag, uint32_t zero) {
    constexpr uint32_t kSegBlocks = kTmaRB / NP;        // blocks of each page per round
    constexpr uint32_t kSegBytesNP = kSegBlocks * 1024u;
    constexpr uint32_t kWarpsPerPage = kTmaCompute / NP;
    extern __shared__ __align__(1024) uint8_t ring[];  // kPairStages x 32 KiB (NP segments)
    __shared__ uint64_t S[2][kTmaRB][8];               // [buf][kSegBlocks * h + block][acc lane]
    __shared__ __align__(8) uint64_t full_bar[kPairStages], empty_bar[kPairStages];
    __shared__ uint64_t sw[24], slast[8], smerge[8], sinit[8];
    if (threadIdx.x < 24) sw[threadIdx.x] = c_xxh.w[threadIdx.x];
    if (threadIdx.x < 8) {
        slast[threadIdx.x] = c_xxh.last[threadIdx.x];
        smerge[threadIdx.x] = c_xxh.merge[threadIdx.x];
        sinit[threadIdx.x] = c_xxh.init[threadIdx.x];
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPairStages; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], kTmaCompute);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t q = 0;  // round counter across this CTA's page groups
    const uint64_t ngroups = (w_hi - w_lo + NP - 1) / NP;
    for (uint64_t t = blockIdx.x; t < ngroups; t += gridDim.x) {
        const uint64_t w0 = w_lo + NP * t;
        PairHalf H[NP];
#pragma unroll
        for (int h = 0; h < NP; ++h) pair_half(regs, big_idx, big_pg, n_big, w0 + h, w_hi, kSegBlocks, H[h]);
        uint32_t rounds = 0;
#pragma unroll
        for (int h = 0; h < NP; ++h) rounds = max(rounds, H[h].rounds);
        if (warp == kTmaCompute + 1) {
            // loader: per round, each active page's segment (bulk copy, or a
            // zero-filled copy by the lanes for a region's partial last page)
            for (uint32_t rr = 0; rr < rounds; ++rr, ++q) {
                const uint32_t st = q % kPairStages, use = q / kPairStages;
                if (use) mbar_wait(&empty_bar[st], (use - 1) & 1);
                uint8_t *dst = ring + (size_t)st * kTmaRound;
                const uint64_t off = (uint64_t)rr * kSegBytesNP;
                int kind[NP];  // 0 idle, 1 bulk copy, 2 zero-filled copy
                bool any_fill = false;
                uint32_t tx = 0;
#pragma unroll
                for (int h = 0; h < NP; ++h) {
                    kind[h] = rr >= H[h].rounds ? 0 : (off + kSegBytesNP <= H[h].len ? 1 : 2);
                    any_fill |= kind[h] == 2;
                    tx += kind[h] == 1 ? kSegBytesNP : 0u;
                }
                if (any_fill) {
#pragma unroll
                    for (int h = 0; h < NP; ++h)
                        if (kind[h] == 2)
                            for (uint32_t o = lane * 16; o < kSegBytesNP; o += 512)
                                *reinterpret_cast<uint4 *>(dst + h * kSegBytesNP + o) =
                                    ld_slot16(H[h].pg, off + o, H[h].len);
                    // order these generic stores before any later bulk copy into the stage
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                __syncwarp();
                if (lane == 0) {
                    if (tx) {
                        mbar_arrive_tx(&full_bar[st], tx);
#pragma unroll
                        for (int h = 0; h < NP; ++h)
                            if (kind[h] == 1) bulk_g2s(dst + h * kSegBytesNP, H[h].pg + off, kSegBytesNP, &full_bar[st]);
                    } else {
                        mbar_arrive(&full_bar[st]);
                    }
                }
            }
        } else if (warp < kTmaCompute) {
            const uint32_t p = lane & 3, b = lane >> 2;
            const uint32_t h = warp / kWarpsPerPage;                 // page of the group
            const uint32_t hb = (warp % kWarpsPerPage) * 8 + b;      // block within the page's segment
            const uint32_t my_rounds = h ? H[1].rounds : H[0].rounds;
            const uint32_t my_bpp = h ? H[1].bpp : H[0].bpp;
            for (uint32_t rr = 0; rr < rounds; ++rr, ++q) {
                const uint32_t st = q % kPairStages, use = q / kPairStages;
                const uint32_t buf = q & 1;
                mbar_wait(&full_bar[st], use & 1);
                uint64_t a0 = 0, a1 = 0;
                if (rr < my_rounds) {
                    const uint8_t *src = ring + (size_t)st * kTmaRound + h * kSegBytesNP + hb * 1024 + p * 16;
                    uint4 d[16];
#pragma unroll
                    for (int s2 = 0; s2 < 16; ++s2) d[s2] = *reinterpret_cast<const uint4 *>(src + s2 * 64);
                    // release once the loads have landed (TMA ring rule)
                    uint32_t fold = 0;
#pragma unroll
                    for (int s2 = 0; s2 < 16; ++s2) fold ^= d[s2].x ^ d[s2].y ^ d[s2].z ^ d[s2].w;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[st] + (fold & zero));
                    const uint32_t bi = rr * kSegBlocks + hb;
#pragma unroll
                    for (int s2 = 0; s2 < 15; ++s2) accum16(a0, a1, d[s2], sw[s2 + 2 * p], sw[s2 + 2 * p + 1]);
                    const bool lastblk = (bi == my_bpp - 1);
                    accum16(a0, a1, d[15], lastblk ? slast[2 * p] : sw[15 + 2 * p],
                            lastblk ? slast[2 * p + 1] : sw[16 + 2 * p]);
                } else {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[st]);
                }
                if (q >= 2) bar_sync(3 + buf, kTmaChainThreads);  // the chain has drained this buffer
                S[buf][h * kSegBlocks + hb][2 * p] = a0;
                S[buf][h * kSegBlocks + hb][2 * p + 1] = a1;
                bar_arrive(1 + buf, kTmaChainThreads);
            }
        } else {
            // chain warp: lanes 8h + l run page h's chain on accumulator lane l
            const uint32_t l = lane & 7, h = (lane >> 3) % NP;
            const uint64_t key = sw[16 + l];
            uint64_t acc = sinit[l];
            const uint32_t hr = h ? H[1].rounds : H[0].rounds;
            const uint32_t hbpp = h ? H[1].bpp : H[0].bpp;
            for (uint32_t rr = 0; rr < rounds; ++rr, ++q) {
                const uint32_t buf = q & 1;
                bar_sync(1 + buf, kTmaChainThreads);
                const uint32_t b0 = rr * kSegBlocks;
                if (rr < hr) {
#pragma unroll 8
                    for (uint32_t j = 0; j < kSegBlocks; ++j) {
                        acc += S[buf][h * kSegBlocks + j][l];
                        if (b0 + j != hbpp - 1) acc = scramble(acc, key);
                    }
                }
                // arrive once the block sums have landed (acc depends on them)
                bar_arrive(3 + buf + (uint32_t)(acc & zero), kTmaChainThreads);
            }
            // merge: r = P * PRIME64_1 + sum_i fold64((acc[2i]^m[2i]) * (acc[2i+1]^m[2i+1]))
            const uint64_t x = acc ^ smerge[l];
            const uint64_t y = __shfl_down_sync(0xffffffffu, x, 1);
            uint64_t m = ((l & 1) == 0) ? ((x * y) ^ __umul64hi(x, y)) : 0;
            m += __shfl_xor_sync(0xffffffffu, m, 2);
            m += __shfl_xor_sync(0xffffffffu, m, 4);
            if ((lane & 7) == 0 && lane < 8 * NP && hr) {
                PairHalf Hh;  // looked up again: keeps P / g / old out of the round loop's registers
                pair_half(regs, big_idx, big_pg, n_big, w0 + h, w_hi, kSegBlocks, Hh);
                uint64_t hv = Hh.P * kP64_1 + m;
                hv ^= hv >> 37;
                hv *= kMx1;
                hv ^= hv >> 32;
                newhash[Hh.g] = hv;
                flags[Hh.g] = (hv != Hh.old) ? tag : 0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// CRUM_VERIFY (restore): recompute XXH3 of every hash-mode slot of the image
// payload and compare with the listed hash.  Warp per slot (P = 4 KiB slots
// use the G = 4 path with the upper half-warp duplicating the lower).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_verify_hash(const DevRegion *__restrict__ regs,
                                                     uint32_t R, const RegStat *__restrict__ rs,
                                                     const uint64_t *__restrict__ hashes,
                                                     const uint8_t *__restrict__ payload, uint64_t K,
                                                     DevStats *st) {
    const uint32_t lane = threadIdx.x & 31;
    __shared__ uint64_t s_w[24];
    stage_secret(s_w);
    __syncthreads();
    LaneKeys k;
    load_lane_keys(k, lane & 3, s_w);
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    for (uint64_t s = (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5); s < K; s += nwarps) {
        // the slot's region is the LAST region whose first slot is <= s
        // (regions listing no slot share `first` with their successor)
        uint32_t lo = 0, hi = R;
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (rs[mid].first <= s) lo = mid; else hi = mid;
        }
        const DevRegion Rg = regs[lo];
        if (Rg.mode != kModeHash) continue;
        const uint64_t P = 1ull << Rg.log2p;
        const uint8_t *slot = payload + rs[lo].payload_base + (s - rs[lo].first) * P;
        const uint32_t bpp = (uint32_t)(P >> 10);
        const uint64_t h = (Rg.log2p == 12) ? xxh3_slot<4, false>(slot, P, bpp, lane, k)
                                            : xxh3_slot<8, false>(slot, P, bpp, lane, k);
        if (lane == 0 && h != hashes[s]) atomicMax(&st->status, (uint32_t)kStCorrupt);
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline int grid_for(uint64_t warps, int sms, int per_sm) {
    uint64_t blocks = (warps + 7) / 8;
    uint64_t cap = (uint64_t)sms * per_sm;
    if (blocks > cap) blocks = cap;
    return blocks ? (int)blocks : 1;
}

void launch_detect_compare(const Launch &L, const DevRegion *regs, const uint32_t *cmp_idx,
                           const uint64_t *cmp_seg, uint32_t n_cmp, uint64_t s_lo, uint64_t s_hi,
                           const uint8_t *force, uint8_t *flags, uint8_t tag) {
    if (s_hi <= s_lo) return;
    k_detect_compare<<<grid_for(s_hi - s_lo, L.sms, 8), 256, 0, L.stream>>>(regs, cmp_idx, cmp_seg, n_cmp, s_lo,
                                                                             s_hi, force, flags, tag);
    ++*L.counter;
}

void launch_detect_hash(const Launch &L, const DevRegion *regs, const uint32_t *hash_idx,
                        const uint64_t *hash_grp, uint32_t n_hash, uint64_t w_lo, uint64_t w_hi,
                        uint8_t *flags, uint64_t *newhash, uint8_t tag) {
    if (w_hi <= w_lo) return;
    k_detect_hash<<<grid_for(w_hi - w_lo, L.sms, 8), 256, 0, L.stream>>>(regs, hash_idx, hash_grp, n_hash, w_lo,
                                                                         w_hi, flags, newhash, tag);
    ++*L.counter;
}

void launch_detect_hash_big(const Launch &L, const DevRegion *regs, const uint32_t *big_idx,
                            const uint64_t *big_pg, uint32_t n_big, uint64_t w_lo, uint64_t w_hi,
                            uint8_t *flags, uint64_t *newhash, uint8_t tag) {
    if (w_hi <= w_lo) return;
    const uint64_t pages = w_hi - w_lo;
    // Page groups only when there are enough pages to give every CTA slot a
    // group: a short range (the host pipeline's first 16 MiB range holds only
    // 8 pages of 2 MiB) finishes sooner with one page per CTA
    if (pages >= (uint64_t)L.sms * kTmaCtasPerSm) {
        const uint64_t cap = (uint64_t)L.sms * kTmaCtasPerSm;
        const size_t smem = (size_t)kPairStages * kTmaRound;
        const uint64_t groups = (pages + NP - 1) / NP;
        const uint64_t per = (groups + cap - 1) / cap;  // balanced: every CTA gets the same number
        const uint64_t grid = (groups + per - 1) / per;
        cudaFuncSetAttribute(k_detect_hash_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_detect_hash_pair<<<(unsigned)grid, kTmaThreads, smem, L.stream>>>(regs, big_idx, big_pg, n_big, w_lo, w_hi,
                                                                            flags, newhash, tag, 0u);
        ++*L.counter;
        return;
    }
    const uint32_t nst = kTmaStages;
    const size_t smem = (size_t)nst * kTmaRound;
    cudaFuncSetAttribute(k_detect_hash_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_detect_hash_tma, kTmaThreads, smem);
    // a page's scramble chain is serial: give every CTA the same number of
    // pages (e.g. 512 x 2 MiB pages -> 256 CTAs x 2, not 444 CTAs x 1-2)
    const uint64_t cap = (uint64_t)L.sms * (uint64_t)std::max(1, std::min(occ, kTmaCtasPerSm));
    const uint64_t per = (pages + cap - 1) / cap;
    const uint64_t blocks = (pages + per - 1) / per;
    k_detect_hash_tma<<<(unsigned)blocks, kTmaThreads, smem, L.stream>>>(regs, big_idx, big_pg, n_big, w_lo, w_hi,
                                                                         flags, newhash, tag, nst);
    ++*L.counter;
}

void launch_verify_hash(const Launch &L, const DevRegion *regs, uint32_t R, const RegStat *rs,
                        const uint64_t *hashes, const uint8_t *payload, uint64_t K, DevStats *st) {
    if (!R || !K) return;
    k_verify_hash<<<L.sms * 4, 256, 0, L.stream>>>(regs, R, rs, hashes, payload, K, st);
    ++*L.counter;
}

}  // namespace crum
