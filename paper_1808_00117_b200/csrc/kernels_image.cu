// kernels_image.cu -- A2 compact, A3 gather + commit, A6 scatter + commit,
// and the v1 image metadata (table, ids, hashes, CRC-32s) on the device.
//
//  * compaction: two passes over the per-page flags (N bytes + N force bytes,
//    uint4 loads, 4096 pages per 256-thread block): per-block counts, then
//    each block sums the counts before it and writes its ids in ascending
//    order (block scan over per-thread counts).  Deterministic: no atomics
//    decide positions.
//  * region stats: one block; per region a binary search of the sorted ids
//    gives (first, n_dirty), then a block scan gives payload/unit offsets.
//  * gather / scatter: one warp per 4 KiB unit of payload, 256-bit loads and
//    stores; the unit -> (region, slot, page) map is a binary search of the
//    per-region unit prefix.  Commit is fused: mirror <- page (compare),
//    table <- new hash (hash), force <- 0.
//  * CRC-32 of the metadata: per-thread 256-byte chunks with a byte table in
//    shared memory, each chunk's raw CRC shifted to its position by a
//    GF(2)[x] multiplication by x^(8*bytes_after) mod P, XOR-reduced.
#include "crum_internal.cuh"

namespace crum {

// ---------------------------------------------------------------------------
// vector helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ld256v(const void *p, uint32_t (&r)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st256(void *p, const uint32_t (&r)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide exclusive scan of one u64 per thread; returns the exclusive
// prefix, *total = block sum.  blockDim.x must be a multiple of 32, <= 1024.
__device__ uint64_t block_excl_scan(uint64_t v, uint64_t *total) {
    __shared__ uint64_t warp_off[32];
    __shared__ uint64_t block_tot;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += t;
    }
    __syncthreads();  // previous call's readers are done with warp_off / block_tot
    if (lane == 31) warp_off[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const uint64_t w = lane < nw ? warp_off[lane] : 0;
        uint64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= (uint32_t)o) wi += t;
        }
        if (lane < nw) warp_off[lane] = wi - w;  // exclusive warp offsets
        if (lane == 31) block_tot = wi;           // lanes >= nw add 0: lane 31 holds the sum
    }
    __syncthreads();
    if (total) *total = block_tot;
    return warp_off[wid] + inc - v;
}

// ---------------------------------------------------------------------------
// A2 compaction
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t thread_dirty_mask(const uint8_t *flags, const uint8_t *force,
                                                      uint64_t base, uint64_t N, int full) {
    if (full) {
        if (base >= N) return 0;
        const uint64_t n = N - base;
        return n >= 16 ? 0xffffu : ((1u << n) - 1);
    }
    const uint4 f = *reinterpret_cast<const uint4 *>(flags + base);
    const uint4 o = *reinterpret_cast<const uint4 *>(force + base);
    const uint32_t w[4] = {f.x | o.x, f.y | o.y, f.z | o.z, f.w | o.w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int b = 0; b < 4; ++b) m |= ((w[i] >> (8 * b)) & 0xffu ? 1u : 0u) << (4 * i + b);
    return m;
}

__global__ void __launch_bounds__(kCompactThreads) k_compact_count(const uint8_t *__restrict__ flags,
                                                                  const uint8_t *__restrict__ force,
                                                                  uint64_t N, int full,
                                                                  uint32_t *__restrict__ blk) {
    const uint64_t base = (uint64_t)blockIdx.x * kPagesPerCompactBlock + threadIdx.x * kPagesPerThread;
    uint32_t c = __popc(thread_dirty_mask(flags, force, base, N, full));
    c = warp_sum(c);
    __shared__ uint32_t s[kCompactThreads / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int i = 0; i < kCompactThreads / 32; ++i) t += s[i];
        blk[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kCompactThreads) k_compact_write(
    const uint8_t *__restrict__ flags, const uint8_t *__restrict__ force, uint64_t N, int full,
    const uint32_t *__restrict__ blk, uint32_t *__restrict__ gids, DevStats *st) {
    // offset of this block = sum of the counts of all earlier blocks
    uint64_t pre = 0;
    for (uint32_t i = threadIdx.x; i < blockIdx.x; i += blockDim.x) pre += blk[i];
    pre = warp_sum(pre);
    __shared__ uint64_t s_pre[kCompactThreads / 32];
    if ((threadIdx.x & 31) == 0) s_pre[threadIdx.x >> 5] = pre;
    __syncthreads();
    uint64_t offset = 0;
    for (int i = 0; i < kCompactThreads / 32; ++i) offset += s_pre[i];

    const uint64_t base = (uint64_t)blockIdx.x * kPagesPerCompactBlock + threadIdx.x * kPagesPerThread;
    uint32_t m = thread_dirty_mask(flags, force, base, N, full);
    uint64_t tot;
    uint64_t pos = offset + block_excl_scan(__popc(m), &tot);
    while (m) {
        const uint32_t b = __ffs(m) - 1;
        gids[pos++] = (uint32_t)(base + b);
        m &= m - 1;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) st->K = offset + tot;
}

void launch_compact(const Launch &L, const uint8_t *flags, const uint8_t *force, uint64_t N, int full,
                    uint32_t *blk_counts, uint32_t *gids, DevStats *st) {
    const uint64_t nblk = (N + kPagesPerCompactBlock - 1) / kPagesPerCompactBlock;
    if (nblk == 0) {
        cudaMemsetAsync(&st->K, 0, sizeof(uint64_t), L.stream);
        return;
    }
    k_compact_count<<<(unsigned)nblk, kCompactThreads, 0, L.stream>>>(flags, force, N, full, blk_counts);
    k_compact_write<<<(unsigned)nblk, kCompactThreads, 0, L.stream>>>(flags, force, N, full, blk_counts,
                                                                      gids, st);
    *L.counter += 2;
}

// ---------------------------------------------------------------------------
// Per-region stats + image header fields (single block).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t *a, uint64_t n, uint64_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if ((uint64_t)a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(1024) k_region_stats(const DevRegion *__restrict__ regs, uint32_t R,
                                                       const uint32_t *__restrict__ gids,
                                                       RegStat *__restrict__ rs, DevStats *st,
                                                       int full, int has_hashes, uint64_t capacity) {
    const uint64_t K = st->K;
    uint64_t carry_pb = 0, carry_u = 0;
    for (uint32_t r0 = 0; r0 < R; r0 += blockDim.x) {
        const uint32_t r = r0 + threadIdx.x;
        uint64_t pb = 0, un = 0, first = 0, nd = 0;
        if (r < R) {
            const DevRegion g = regs[r];
            first = lower_bound_u32(gids, K, g.page_base);
            nd = lower_bound_u32(gids, K, g.page_base + g.n_pages) - first;
            pb = nd << g.log2p;
            un = nd << (g.log2p - kSegLog2);
        }
        uint64_t tpb, tun;
        const uint64_t epb = block_excl_scan(pb, &tpb);
        const uint64_t eun = block_excl_scan(un, &tun);
        if (r < R) {
            rs[r].first = first;
            rs[r].n_dirty = nd;
            rs[r].payload_base = carry_pb + epb;
            rs[r].unit_base = carry_u + eun;
        }
        carry_pb += tpb;
        carry_u += tun;
    }
    if (threadIdx.x == 0) {
        const uint64_t meta = 64 + 48ull * R + round_up(4 * K, 8) + (has_hashes ? 8 * K : 0);
        const uint64_t poff = round_up(meta, 4096);
        st->meta_bytes = meta;
        st->poff = poff;
        st->payload_bytes = carry_pb;
        st->total_units = carry_u;
        st->image_bytes = poff + carry_pb;
        st->capacity = capacity;
        st->status = (poff + carry_pb > capacity) ? kStCapacity : kStOk;
        st->img_flags = (full ? 1u : 0u) | (has_hashes ? 2u : 0u);
        st->n_regions = R;
        st->dirty_bytes = 0;
        st->dirty_runs = 0;
        st->crc_acc = 0;
    }
}

void launch_region_stats(const Launch &L, const DevRegion *regs, uint32_t R, const uint32_t *gids,
                         RegStat *rs, DevStats *st, int full, int has_hashes, uint64_t capacity) {
    k_region_stats<<<1, 1024, 0, L.stream>>>(regs, R, gids, rs, st, full, has_hashes, capacity);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// Image metadata: region table, ids, hash list, zero padding; dirty bytes and
// runs of the listed pages.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t region_of_page(const DevRegion *regs, uint32_t R, uint64_t g) {
    uint32_t lo = 0, hi = R;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (regs[mid].page_base <= g) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_meta(const DevRegion *__restrict__ regs, uint32_t R,
                                              const uint32_t *__restrict__ gids,
                                              const uint64_t *__restrict__ newhash,
                                              const RegStat *__restrict__ rs, DevStats *st,
                                              uint8_t *__restrict__ img) {
    if (st->status != kStOk) return;
    const uint64_t K = st->K;
    const bool has_hashes = (st->img_flags & 2u) != 0;
    const uint64_t meta = st->meta_bytes, poff = st->poff;
    uint32_t *ids = reinterpret_cast<uint32_t *>(img + 64 + 48ull * R);
    uint64_t *hashes = reinterpret_cast<uint64_t *>(img + 64 + 48ull * R + round_up(4 * K, 8));
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t r = tid; r < R; r += nth) {
        const DevRegion g = regs[r];
        uint8_t *e = img + 64 + 48 * r;
        reinterpret_cast<uint32_t *>(e)[0] = g.id;
        reinterpret_cast<uint32_t *>(e)[1] = g.mode;
        reinterpret_cast<uint64_t *>(e)[1] = g.bytes;
        reinterpret_cast<uint64_t *>(e)[2] = 1ull << g.log2p;
        reinterpret_cast<uint64_t *>(e)[3] = g.n_pages;
        reinterpret_cast<uint64_t *>(e)[4] = rs[r].n_dirty;
        reinterpret_cast<uint64_t *>(e)[5] = rs[r].first;
    }
    uint64_t dbytes = 0, runs = 0;
    for (uint64_t k = tid; k < K; k += nth) {
        const uint64_t gid = gids[k];
        const uint32_t r = region_of_page(regs, R, gid);
        const DevRegion g = regs[r];
        const uint64_t i = gid - g.page_base;
        ids[k] = (uint32_t)i;
        if (has_hashes) hashes[k] = (g.mode == kModeHash) ? newhash[gid] : 0;
        dbytes += min((uint64_t)1 << g.log2p, (uint64_t)(g.bytes - (i << g.log2p)));
        runs += (k == rs[r].first || gids[k - 1] + 1 != gid) ? 1 : 0;
    }
    if (tid == 0 && (K & 1)) ids[K] = 0;
    for (uint64_t b = meta + tid; b < poff; b += nth) img[b] = 0;
    dbytes = warp_sum(dbytes);
    runs = warp_sum(runs);
    if ((threadIdx.x & 31) == 0 && (dbytes | runs)) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&st->dirty_bytes), (unsigned long long)dbytes);
        atomicAdd(reinterpret_cast<unsigned long long *>(&st->dirty_runs), (unsigned long long)runs);
    }
}

void launch_meta(const Launch &L, const DevRegion *regs, uint32_t R, const uint32_t *gids,
                 const uint64_t *newhash, const RegStat *rs, DevStats *st, uint8_t *img) {
    k_meta<<<L.sms * 2, 256, 0, L.stream>>>(regs, R, gids, newhash, rs, st, img);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// A3 gather + commit (img == nullptr: commit only, i.e. crum_sync_shadow).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t region_of_unit(const RegStat *rs, uint32_t R, uint64_t u) {
    uint32_t lo = 0, hi = R;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (rs[mid].unit_base <= u) lo = mid; else hi = mid;
    }
    return lo;
}

// Copy one 4 KiB unit: `len` logical bytes from src (rest zero) to dst_a
// (full 4 KiB, may be null) and the first `len` bytes to dst_b (may be null).
__device__ __forceinline__ void copy_unit(const uint8_t *src, uint64_t len, bool aligned32,
                                          uint8_t *dst_a, uint8_t *dst_b, uint32_t lane) {
    if (len >= kSegBytes && aligned32) {
        uint32_t v[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) ld256v(src + i * 1024 + lane * 32, v[i]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (dst_a) st256(dst_a + i * 1024 + lane * 32, v[i]);
            if (dst_b) st256(dst_b + i * 1024 + lane * 32, v[i]);
        }
    } else if (len >= kSegBytes) {
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = *reinterpret_cast<const uint4 *>(src + i * 512 + lane * 16);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (dst_a) *reinterpret_cast<uint4 *>(dst_a + i * 512 + lane * 16) = v[i];
            if (dst_b) *reinterpret_cast<uint4 *>(dst_b + i * 512 + lane * 16) = v[i];
        }
    } else if (len == 0) {
        if (dst_a) {
            const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4 *>(dst_a + i * 512 + lane * 16) = z;
        }
    } else {
        for (uint32_t o = lane; o < kSegBytes; o += 32) {
            const uint8_t v = o < len ? src[o] : 0;
            if (dst_a) dst_a[o] = v;
            if (dst_b && o < len) dst_b[o] = v;
        }
    }
}

__global__ void __launch_bounds__(256) k_gather(const DevRegion *__restrict__ regs, uint32_t R,
                                                const uint32_t *__restrict__ gids,
                                                const uint64_t *__restrict__ newhash,
                                                const RegStat *__restrict__ rs,
                                                const DevStats *__restrict__ st,
                                                uint8_t *__restrict__ dst_base, uint64_t dst_unit0,
                                                int add_poff, uint8_t *__restrict__ force,
                                                uint64_t unit_lo, uint64_t unit_hi) {
    if (st->status != kStOk) return;
    const uint64_t hi = min(unit_hi, st->total_units);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    uint8_t *payload = dst_base ? dst_base + (add_poff ? st->poff : 0) : nullptr;
    for (uint64_t u = unit_lo + (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5); u < hi; u += nwarps) {
        const uint32_t r = region_of_unit(rs, R, u);
        const DevRegion g = regs[r];
        const RegStat s = rs[r];
        const uint32_t sh = g.log2p - kSegLog2;
        const uint64_t ru = u - s.unit_base;
        const uint64_t j = ru >> sh, seg = ru & ((1ull << sh) - 1);
        const uint64_t gid = gids[s.first + j];
        const uint64_t i = gid - g.page_base;
        const uint64_t off = (i << g.log2p) + (seg << kSegLog2);
        const uint64_t len = g.bytes > off ? min((uint64_t)kSegBytes, g.bytes - off) : 0;
        // payload byte offset of unit u is u * 4096 (slots are whole 4 KiB units)
        uint8_t *dst_img = payload ? payload + ((u - dst_unit0) << kSegLog2) : nullptr;
        uint8_t *dst_mir = (g.mode == kModeCompare) ? g.mirror + off : nullptr;
        if (dst_img || dst_mir) copy_unit(g.base + off, len, g.aligned32 != 0, dst_img, dst_mir, lane);
        if (seg == 0 && lane == 0) {
            if (g.mode == kModeHash) g.table[i] = newhash[gid];
            force[gid] = 0;
        }
    }
}

void launch_gather(const Launch &L, const DevRegion *regs, uint32_t R, const uint32_t *gids,
                   const uint64_t *newhash, const RegStat *rs, const DevStats *st, uint8_t *dst_base,
                   uint64_t dst_unit0, int add_poff, uint8_t *force, uint64_t unit_lo, uint64_t unit_hi) {
    if (unit_hi <= unit_lo || !R) return;
    uint64_t blocks = (unit_hi - unit_lo + 7) / 8;
    const uint64_t cap = (uint64_t)L.sms * 8;
    if (blocks > cap) blocks = cap;
    k_gather<<<(unsigned)blocks, 256, 0, L.stream>>>(regs, R, gids, newhash, rs, st, dst_base, dst_unit0,
                                                     add_poff, force, unit_lo, unit_hi);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// CRC-32 (zlib) of the metadata [64, meta_bytes) and the header.
// ---------------------------------------------------------------------------
struct X2N {
    uint32_t t[32];  // x^(2^k) mod P, reflected
};

__device__ __forceinline__ uint32_t gf2_mulmod(uint32_t a, uint32_t b) {
    // reflected GF(2)[x] product mod the CRC-32 polynomial (loop ends at the
    // lowest set bit of a, so a == 0 must be handled up front)
    if (a == 0) return 0;
    uint32_t m = 0x80000000u, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
}

__device__ __forceinline__ uint32_t xpow8n(uint64_t n, const uint32_t *x2n) {
    // x^(8n) mod P
    uint32_t p = 0x80000000u;
    uint32_t k = 3;
    while (n) {
        if (n & 1) p = gf2_mulmod(x2n[k & 31], p);
        n >>= 1;
        ++k;
    }
    return p;
}

constexpr uint32_t kCrcChunk = 256;

__global__ void __launch_bounds__(256) k_crc_meta(const uint8_t *__restrict__ img, DevStats *st,
                                                  X2N x2n) {
    if (st->status != kStOk) return;
    __shared__ uint32_t T[256];
    __shared__ uint32_t sx[32];
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
        T[i] = c;
    }
    if (threadIdx.x < 32) sx[threadIdx.x] = x2n.t[threadIdx.x];
    __syncthreads();
    const uint64_t len = st->meta_bytes - 64;
    const uint8_t *data = img + 64;
    const uint64_t nchunks = (len + kCrcChunk - 1) / kCrcChunk;
    uint32_t acc = 0;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
         c += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b0 = c * kCrcChunk, b1 = min(len, b0 + kCrcChunk);
        uint32_t raw = 0;
        for (uint64_t b = b0; b < b1; ++b) raw = T[(raw ^ data[b]) & 0xffu] ^ (raw >> 8);
        acc ^= gf2_mulmod(xpow8n(len - b1, sx), raw);  // first operand is never 0
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicXor(&st->crc_acc, acc);
}

void launch_crc_meta(const Launch &L, const uint8_t *img, DevStats *st, const uint32_t *x2n) {
    X2N x;
    for (int i = 0; i < 32; ++i) x.t[i] = x2n[i];
    k_crc_meta<<<L.sms * 2, 256, 0, L.stream>>>(img, st, x);
    ++*L.counter;
}

__device__ __forceinline__ void put32(uint8_t *p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
__device__ __forceinline__ void put64(uint8_t *p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

__global__ void k_header(uint8_t *img, DevStats *st, X2N x2n) {
    if (st->status != kStOk) return;
    const uint64_t len = st->meta_bytes - 64;
    const uint32_t meta_crc = st->crc_acc ^ gf2_mulmod(0xffffffffu, xpow8n(len, x2n.t)) ^ 0xffffffffu;
    st->meta_crc = meta_crc;
    uint8_t h[64];
    h[0] = 'C'; h[1] = 'R'; h[2] = 'U'; h[3] = 'M';
    put32(h + 4, 1);
    put32(h + 8, st->img_flags);
    put32(h + 12, st->n_regions);
    put64(h + 16, st->K);
    put64(h + 24, st->meta_bytes);
    put64(h + 32, st->poff);
    put64(h + 40, st->payload_bytes);
    put32(h + 48, meta_crc);
    put64(h + 52, 0);
    uint32_t c = 0xffffffffu;
    for (int i = 0; i < 60; ++i) {
        c ^= h[i];
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    put32(h + 60, c ^ 0xffffffffu);
    for (int i = 0; i < 64; ++i) img[i] = h[i];
}

void launch_header(const Launch &L, uint8_t *img, DevStats *st, const uint32_t *x2n) {
    X2N x;
    for (int i = 0; i < 32; ++i) x.t[i] = x2n[i];
    k_header<<<1, 1, 0, L.stream>>>(img, st, x);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// A6 restore: validation of the id list, then scatter + commit.
// rs[] here comes from the image's region table (validated on the host).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t region_of_slot(const RegStat *rs, uint32_t R, uint64_t k) {
    uint32_t lo = 0, hi = R;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (rs[mid].first <= k) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_restore_validate(const DevRegion *__restrict__ regs, uint32_t R,
                                                          const RegStat *__restrict__ rs,
                                                          const uint8_t *__restrict__ img,
                                                          DevStats *st) {
    const uint64_t K = st->K;
    const bool has_hashes = (st->img_flags & 2u) != 0;
    const uint32_t *ids = reinterpret_cast<const uint32_t *>(img + 64 + 48ull * R);
    const uint64_t *hashes = reinterpret_cast<const uint64_t *>(img + 64 + 48ull * R + round_up(4 * K, 8));
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    uint32_t bad = 0;
    uint64_t dbytes = 0, runs = 0;
    for (uint64_t k = tid; k < K; k += nth) {
        const uint32_t r = region_of_slot(rs, R, k);
        const DevRegion g = regs[r];
        const uint64_t i = ids[k];
        const bool first = (k == rs[r].first);
        if (i >= g.n_pages) bad = 1;
        if (!first && ids[k - 1] >= i) bad = 1;
        if (has_hashes && g.mode == kModeCompare && hashes[k] != 0) bad = 1;
        if (i < g.n_pages) dbytes += min((uint64_t)1 << g.log2p, (uint64_t)(g.bytes - (i << g.log2p)));
        runs += (first || ids[k - 1] + 1 != i) ? 1 : 0;
    }
    bad = __any_sync(0xffffffffu, bad);
    dbytes = warp_sum(dbytes);
    runs = warp_sum(runs);
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicMax(&st->status, (uint32_t)kStCorrupt);
        if (dbytes | runs) {
            atomicAdd(reinterpret_cast<unsigned long long *>(&st->dirty_bytes), (unsigned long long)dbytes);
            atomicAdd(reinterpret_cast<unsigned long long *>(&st->dirty_runs), (unsigned long long)runs);
        }
    }
}

void launch_restore_validate(const Launch &L, const DevRegion *regs, uint32_t R, const RegStat *rs,
                             const uint8_t *img, DevStats *st) {
    if (!R) return;
    k_restore_validate<<<L.sms * 2, 256, 0, L.stream>>>(regs, R, rs, img, st);
    ++*L.counter;
}

__global__ void __launch_bounds__(256) k_scatter(const DevRegion *__restrict__ regs, uint32_t R,
                                                 const RegStat *__restrict__ rs,
                                                 const uint8_t *__restrict__ meta,
                                                 const DevStats *__restrict__ st,
                                                 const uint8_t *__restrict__ src_base, uint64_t src_unit0,
                                                 int add_poff, uint8_t *__restrict__ force,
                                                 uint64_t unit_lo, uint64_t unit_hi) {
    if (st->status != kStOk) return;
    const uint64_t K = st->K;
    const uint32_t *ids = reinterpret_cast<const uint32_t *>(meta + 64 + 48ull * R);
    const uint64_t *hashes = reinterpret_cast<const uint64_t *>(meta + 64 + 48ull * R + round_up(4 * K, 8));
    const uint8_t *payload = src_base + (add_poff ? st->poff : 0);
    const uint64_t hi = min(unit_hi, st->total_units);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    for (uint64_t u = unit_lo + (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5); u < hi; u += nwarps) {
        const uint32_t r = region_of_unit(rs, R, u);
        const DevRegion g = regs[r];
        const RegStat s = rs[r];
        const uint32_t sh = g.log2p - kSegLog2;
        const uint64_t ru = u - s.unit_base;
        const uint64_t j = ru >> sh, seg = ru & ((1ull << sh) - 1);
        const uint64_t k = s.first + j;
        const uint64_t i = ids[k];
        const uint64_t off = (i << g.log2p) + (seg << kSegLog2);
        if (g.bytes > off) {
            const uint64_t len = min((uint64_t)kSegBytes, g.bytes - off);
            const uint8_t *src = payload + ((u - src_unit0) << kSegLog2);
            uint8_t *dst_mir = (g.mode == kModeCompare) ? g.mirror + off : nullptr;
            if (len == kSegBytes) {
                copy_unit(src, len, g.aligned32 != 0, g.base + off, dst_mir, lane);
            } else {
                for (uint32_t o = lane; o < len; o += 32) {
                    g.base[off + o] = src[o];
                    if (dst_mir) dst_mir[o] = src[o];
                }
            }
        }
        if (seg == 0 && lane == 0) {
            if (g.mode == kModeHash) g.table[i] = hashes[k];
            force[g.page_base + i] = 0;
        }
    }
}

void launch_scatter(const Launch &L, const DevRegion *regs, uint32_t R, const RegStat *rs,
                    const uint8_t *meta, const DevStats *st, const uint8_t *src_base, uint64_t src_unit0,
                    int add_poff, uint8_t *force, uint64_t unit_lo, uint64_t unit_hi) {
    if (unit_hi <= unit_lo || !R) return;
    uint64_t blocks = (unit_hi - unit_lo + 7) / 8;
    const uint64_t cap = (uint64_t)L.sms * 8;
    if (blocks > cap) blocks = cap;
    k_scatter<<<(unsigned)blocks, 256, 0, L.stream>>>(regs, R, rs, meta, st, src_base, src_unit0, add_poff,
                                                      force, unit_lo, unit_hi);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// debug: flags | force, global page order
// ---------------------------------------------------------------------------
__global__ void k_export_flags(const uint8_t *flags, const uint8_t *force, uint64_t N, uint8_t *out) {
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < N;
         g += (uint64_t)gridDim.x * blockDim.x)
        out[g] = (flags[g] | force[g]) ? 1 : 0;
}

void launch_export_flags(const Launch &L, const uint8_t *flags, const uint8_t *force, uint64_t N,
                         uint8_t *out) {
    if (!N) return;
    k_export_flags<<<L.sms * 4, 256, 0, L.stream>>>(flags, force, N, out);
    ++*L.counter;
}

}  // namespace crum
