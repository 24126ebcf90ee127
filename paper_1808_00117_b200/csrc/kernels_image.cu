// kernels_image.cu -- A2 compact, A3 gather + commit, A6 scatter + commit,
// and the v1 image metadata (table, ids, hashes, CRC-32s) on the device.
//
//  * compaction (per page range [p_lo, p_hi), ranges in ascending order):
//    two passes over the per-page flags (uint4 loads, 4096 pages per
//    256-thread block).  Pass 1: per-block (count, 4 KiB units).  Pass 2: each
//    block sums the totals of the blocks before it (plus the running totals
//    of earlier ranges), block-scans (count, units) over its threads and
//    writes, per dirty page in ascending order: the global page id, the
//    slot's payload unit offset, the region-local id and (hash regions) the
//    new hash; per-region counts, runs and dirty bytes accumulate with
//    integer atomics (order-free, deterministic).  Positions are decided by
//    scans only -- the image is canonical.  The last block to finish (done
//    counter) publishes the running totals and, for the final range, the
//    per-region prefix sums, the header fields and the region table.
//  * gather / scatter: one warp per 8 consecutive 4 KiB payload units, one
//    binary search per task, 256-bit loads and stores; commit fused.
//  * CRC-32 of table || ids || hashes: per-thread 64-byte chunks (byte table
//    in shared memory; zlib's ~0 init folded into chunk 0), each chunk's raw
//    CRC shifted to its position by a GF(2)[x] product with x^(8*after) mod
//    P, XOR-reduced; the last block finalises and writes the header.  The
//    kernel also copies ids/hashes from scratch into the image tail.
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// A2 compaction
// ---------------------------------------------------------------------------
// Dirty mask of this thread's 16 pages [base, base+16) within [p_lo, p_hi).
__device__ __forceinline__ uint32_t thread_mask(const CompactArgs &a, uint64_t base) {
    uint32_t m = 0;
    if (base >= a.p_hi) return 0;  // nothing of ours in range (also keeps loads in bounds)
    if (a.full) {
#pragma unroll
        for (int b = 0; b < 16; ++b) m |= (base + b >= a.p_lo && base + b < a.p_hi ? 1u : 0u) << b;
        return m;
    }
    const uint4 f = *reinterpret_cast<const uint4 *>(a.flags + base);
    const uint4 o = *reinterpret_cast<const uint4 *>(a.force + base);
    const uint32_t fw[4] = {f.x, f.y, f.z, f.w}, ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t fb = (fw[i] >> (8 * b)) & 0xffu, ob = (ow[i] >> (8 * b)) & 0xffu;
            const uint64_t g = base + 4 * i + b;
            m |= ((fb == a.tag || ob != 0) && g >= a.p_lo && g < a.p_hi ? 1u : 0u) << (4 * i + b);
        }
    return m;
}

// 4 KiB units of the dirty pages in mask (pages advance through regions).
__device__ __forceinline__ uint64_t mask_units(const CompactArgs &a, uint64_t base, uint32_t m) {
    if (!m) return 0;
    uint32_t r = region_of_page(a.regs, a.R, base + (__ffs(m) - 1));
    uint64_t next = (r + 1 < a.R) ? a.regs[r + 1].page_base : ~0ull;
    uint32_t sh = a.regs[r].log2p - kSegLog2;
    uint64_t u = 0;
    while (m) {
        const uint64_t g = base + (__ffs(m) - 1);
        while (g >= next) {
            ++r;
            next = (r + 1 < a.R) ? a.regs[r + 1].page_base : ~0ull;
            sh = a.regs[r].log2p - kSegLog2;
        }
        u += 1ull << sh;
        m &= m - 1;
    }
    return u;
}

__device__ void compact_finalize(const CompactArgs &a, uint64_t K, uint64_t U) {
    // per-region prefix sums (first slot, payload offset, unit offset) + table
    uint64_t carry_first = 0, carry_units = 0;
    for (uint32_t r0 = 0; r0 < a.R; r0 += blockDim.x) {
        const uint32_t r = r0 + threadIdx.x;
        uint64_t nd = 0, un = 0;
        DevRegion g{};
        if (r < a.R) {
            g = a.regs[r];
            nd = *(volatile uint32_t *)(a.reg_nd + r);
            un = nd << (g.log2p - kSegLog2);
        }
        uint64_t tn, tun;
        const uint64_t en = block_excl_scan(nd, &tn);
        const uint64_t eun = block_excl_scan(un, &tun);
        if (r < a.R) {
            RegStat s;
            s.first = carry_first + en;
            s.n_dirty = nd;
            s.unit_base = carry_units + eun;
            s.payload_base = s.unit_base << kSegLog2;
            a.rs[r] = s;
            if (a.head) {
                uint8_t *e = a.head + 64 + 48ull * r;
                reinterpret_cast<uint32_t *>(e)[0] = g.id;
                reinterpret_cast<uint32_t *>(e)[1] = g.mode;
                reinterpret_cast<uint64_t *>(e)[1] = g.bytes;
                reinterpret_cast<uint64_t *>(e)[2] = 1ull << g.log2p;
                reinterpret_cast<uint64_t *>(e)[3] = g.n_pages;
                reinterpret_cast<uint64_t *>(e)[4] = nd;
                reinterpret_cast<uint64_t *>(e)[5] = s.first;
            }
        }
        carry_first += tn;
        carry_units += tun;
    }
    const uint64_t poff = round_up(64 + 48ull * a.R, 4096);
    const uint64_t payload = U << kSegLog2;
    (void)carry_units;
    const uint64_t ids_off = poff + payload;
    const uint64_t image = ids_off + round_up(4 * K, 8) + (a.has_hashes ? 8 * K : 0);
    if (a.head)
        for (uint64_t b = 64 + 48ull * a.R + threadIdx.x; b < poff; b += blockDim.x) a.head[b] = 0;
    if (threadIdx.x == 0) {
        DevStats *st = a.st;
        st->K = K;
        st->total_units = U;
        st->poff = poff;
        st->payload_bytes = payload;
        st->ids_off = ids_off;
        st->image_bytes = image;
        st->capacity = a.capacity;
        st->status = image > a.capacity ? kStCapacity : kStOk;
        st->img_flags = (a.full ? 1u : 0u) | (a.has_hashes ? 2u : 0u);
        st->n_regions = a.R;
    }
}

constexpr uint32_t kRegAgg = 64;  // per-block region counters kept in shared memory

// Unit -> slot map entries of pages with more than 2^kU2sDirectLog2 units
// (128 KiB and larger pages).  Smaller pages are written inline by their
// thread.  The threads that own large dirty pages are listed in shared memory
// and the block's warps take them in turn: a warp walks the owner's dirty
// pages in lock step (same region lookups) and stores each large page's
// entries lane-strided.  (One thread storing a 2 MiB page's 512 entries made
// compaction of 2 MiB pages 52 us; one warp per owning thread still left
// the 512-page C2 case -- all pages owned by warp 0 -- at 12 us of 22.)
// Call with every thread of the block.
struct U2sSmem {
    uint32_t n;
    uint16_t who[kCompactThreads];
    uint32_t m[kCompactThreads];
    uint64_t pos[kCompactThreads], upos[kCompactThreads];
};

__device__ __forceinline__ void u2s_fill_big(const CompactArgs &a, uint64_t base, uint32_t m0, uint64_t pos0,
                                             uint64_t upos0, bool has_big, U2sSmem &sm) {
    if (threadIdx.x == 0) sm.n = 0;
    __syncthreads();
    if (has_big) {
        const uint32_t i = atomicAdd(&sm.n, 1u);
        sm.who[i] = (uint16_t)threadIdx.x;
        sm.m[threadIdx.x] = m0;
        sm.pos[threadIdx.x] = pos0;
        sm.upos[threadIdx.x] = upos0;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const uint64_t blk_base = base - (uint64_t)threadIdx.x * kPagesPerThread;
    for (uint32_t i = threadIdx.x >> 5; i < sm.n; i += nw) {
        const uint32_t t = sm.who[i];
        uint32_t mm = sm.m[t];
        uint64_t pos = sm.pos[t], upos = sm.upos[t];
        const uint64_t b0 = blk_base + (uint64_t)t * kPagesPerThread;
        uint32_t r = region_of_page(a.regs, a.R, b0 + (__ffs(mm) - 1));
        uint32_t l2 = a.regs[r].log2p;
        uint64_t next = (r + 1 < a.R) ? a.regs[r + 1].page_base : ~0ull;
        while (mm) {
            const uint64_t gid = b0 + (__ffs(mm) - 1);
            while (gid >= next) {
                ++r;
                l2 = a.regs[r].log2p;
                next = (r + 1 < a.R) ? a.regs[r + 1].page_base : ~0ull;
            }
            const uint32_t n = 1u << (l2 - kSegLog2);
            if (l2 - kSegLog2 > kU2sDirectLog2)
                for (uint32_t j = lane; j < n; j += 32) a.u2s[upos + j] = (uint32_t)pos;
            ++pos;
            upos += n;
            mm &= mm - 1;
        }
    }
}


// ---------------------------------------------------------------------------
// A2 in one pass (default): the blocks take logical ids from a ticket, publish
// their (pages, units) aggregates in 64-bit status words and find their
// exclusive prefix by decoupled look-back (so a block never waits on one that
// has not started), then write ids, unit offsets and the unit->slot map in order.
// Status word: [63:62] 1 aggregate / 2 inclusive prefix, [61:31] pages,
// [30:0] 4 KiB units.  The words (blk_units reinterpreted) and the ticket
// (done[2]) are reset by the last block, so every launch starts from zero.
// On the first range logical block 0 zeroes the per-call accumulators before
// it publishes; every other block touches them only after its look-back.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t cpack(uint64_t flag, uint64_t cnt, uint64_t units) {
    return (flag << 62) | ((cnt & 0x7fffffffull) << 31) | (units & 0x7fffffffull);
}
__device__ __forceinline__ void st_rel64(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acq64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kCompactThreads) k_compact_onepass(CompactArgs a) {
    __shared__ U2sSmem s_u2s;
    __shared__ uint64_t s_off[2];
    __shared__ uint32_t s_blk;
    __shared__ bool s_last;
    __shared__ uint32_t s_rcnt[kRegAgg];
    __shared__ uint32_t s_r0;
    uint64_t *status = a.blk_units;
    uint32_t *ticket = a.done + 2;
    // running totals of earlier ranges: loaded up front (thread 0 uses them
    // after the look-back), so the load overlaps the ticket and the scans
    // (a single-block launch needs no ticket, fence or last-block election)
    __shared__ uint64_t s_rb[2];
    const bool single = gridDim.x == 1;
    RangeTotals rb0{};
    if (threadIdx.x == 0) {
        rb0 = a.rb[a.c];
        s_rb[0] = rb0.k;
        s_rb[1] = rb0.units;
        s_blk = single ? 0u : atomicAdd(ticket, 1u);
    }
    if (threadIdx.x < kRegAgg) s_rcnt[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t blk = s_blk;
    if (threadIdx.x == 0) s_r0 = region_of_page(a.regs, a.R, a.p_lo + (uint64_t)blk * kPagesPerCompactBlock);
    if (a.first_range && blk == 0) {
        for (uint32_t r = threadIdx.x; r < a.R; r += blockDim.x) a.reg_nd[r] = 0;
        if (threadIdx.x == 0) {
            a.st->dirty_bytes = 0;
            a.st->dirty_runs = 0;
            a.st->crc_acc = 0;
            a.st->status = kStOk;
        }
        __threadfence();
    }
    const uint64_t base = a.p_lo + (uint64_t)blk * kPagesPerCompactBlock + threadIdx.x * kPagesPerThread;
    uint32_t m = thread_mask(a, base);
    if (base < a.p_hi) {  // consume this range's detect marks (flags are zero between calls)
        if (base >= a.p_lo && base + kPagesPerThread <= a.p_hi) {
            *reinterpret_cast<uint4 *>(a.flags + base) = make_uint4(0, 0, 0, 0);
        } else {
            for (uint32_t b = 0; b < kPagesPerThread; ++b)
                if (base + b >= a.p_lo && base + b < a.p_hi) a.flags[base + b] = 0;
        }
    }
    uint64_t tc, tu;
    const uint64_t ec = block_excl_scan(__popc(m), &tc);
    const uint64_t eu = block_excl_scan(mask_units(a, base, m), &tu);  // syncs: s_r0 visible
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        uint64_t pc = 0, pu = 0;
        if (blk == 0) {
            if (lane == 0) st_rel64(status, cpack(2, tc, tu));
        } else {
            if (lane == 0) st_rel64(status + blk, cpack(1, tc, tu));
            int64_t top = (int64_t)blk - 1;
            while (top >= 0) {
                const int64_t idx = top - (int64_t)lane;
                uint64_t v = cpack(2, 0, 0);  // before block 0: prefix 0
                uint32_t flag = 2;
                if (idx >= 0) {
                    do {
                        v = ld_acq64(status + idx);
                        flag = (uint32_t)(v >> 62);
                    } while (flag == 0);
                }
                const uint32_t pm = __ballot_sync(0xffffffffu, flag == 2);
                const int first = pm ? __ffs(pm) - 1 : 32;
                const uint64_t c = ((int)lane <= first) ? ((v >> 31) & 0x7fffffffull) : 0;
                const uint64_t u = ((int)lane <= first) ? (v & 0x7fffffffull) : 0;
                pc += warp_sum(c);
                pu += warp_sum(u);
                if (pm) break;
                top -= 32;
            }
            if (lane == 0) st_rel64(status + blk, cpack(2, pc + tc, pu + tu));
        }
        if (lane == 0) {
            s_off[0] = rb0.k + pc;
            s_off[1] = rb0.units + pu;
        }
    }
    __syncthreads();
    uint64_t pos = s_off[0] + ec, upos = s_off[1] + eu;
    const uint32_t m0 = m;
    bool has_big = false;
    const uint64_t pos0 = pos, upos0 = upos;
    uint64_t dbytes = 0;
    if (m) {
        uint32_t r = region_of_page(a.regs, a.R, base + (__ffs(m) - 1));
        DevRegion g = a.regs[r];
        uint64_t next = (r + 1 < a.R) ? a.regs[r + 1].page_base : ~0ull;
        uint32_t cnt = 0;
        while (m) {
            const int b = __ffs(m) - 1;
            const uint64_t gid = base + b;
            while (gid >= next) {
                if (cnt) {
                    if (r - s_r0 < kRegAgg) atomicAdd(&s_rcnt[r - s_r0], cnt);
                    else atomicAdd(a.reg_nd + r, cnt);
                }
                cnt = 0;
                ++r;
                g = a.regs[r];
                next = (r + 1 < a.R) ? a.regs[r + 1].page_base : ~0ull;
            }
            const uint64_t i = gid - g.page_base;
            a.gids[pos] = (uint32_t)gid;
            a.sunit[pos] = upos;
            if (g.log2p - kSegLog2 > kU2sDirectLog2) has_big = true;
            else
                for (uint32_t j = 0; j < (1u << (g.log2p - kSegLog2)); ++j) a.u2s[upos + j] = (uint32_t)pos;
            a.lids[pos] = (uint32_t)i;
            if (a.has_hashes) a.lhash[pos] = (g.mode == kModeHash) ? a.newhash[gid] : 0;
            dbytes += page_len(g, i);
            ++cnt;
            ++pos;
            upos += 1ull << (g.log2p - kSegLog2);
            m &= m - 1;
        }
        if (cnt) {
            if (r - s_r0 < kRegAgg) atomicAdd(&s_rcnt[r - s_r0], cnt);
            else atomicAdd(a.reg_nd + r, cnt);
        }
    }
    u2s_fill_big(a, base, m0, pos0, upos0, has_big, s_u2s);
    __syncthreads();
    if (threadIdx.x < kRegAgg && s_rcnt[threadIdx.x] && s_r0 + threadIdx.x < a.R)
        atomicAdd(a.reg_nd + s_r0 + threadIdx.x, s_rcnt[threadIdx.x]);
    dbytes = warp_sum(dbytes);
    if ((threadIdx.x & 31) == 0 && dbytes)
        atomicAdd(reinterpret_cast<unsigned long long *>(&a.st->dirty_bytes), (unsigned long long)dbytes);
    // ---- last block: totals, reset of the look-back state, finalise ----
    if (!single) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = (atomicAdd(a.done, 1u) == gridDim.x - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
    } else {
        __syncthreads();  // this block's region counts and bytes are in
    }
    // inclusive prefix of the last block
    const uint64_t vlast = single ? cpack(2, tc, tu) : ld_acq64(status + gridDim.x - 1);
    const uint64_t K = s_rb[0] + ((vlast >> 31) & 0x7fffffffull);
    const uint64_t U = s_rb[1] + (vlast & 0x7fffffffull);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) status[i] = 0;
    if (threadIdx.x == 0) {
        a.rb[a.c + 1].k = K;
        a.rb[a.c + 1].units = U;
        if (a.rb_host) {
            volatile RangeTotals *h = a.rb_host + a.c + 1;
            h->k = K;
            h->units = U;
        }
        *a.done = 0;
        *ticket = 0;
    }
    if (a.final_range) compact_finalize(a, K, U);
}

void launch_compact(const Launch &L, const CompactArgs &a) {
    uint64_t nblk = a.p_hi > a.p_lo ? (a.p_hi - a.p_lo + kPagesPerCompactBlock - 1) / kPagesPerCompactBlock : 0;
    if (nblk == 0) nblk = 1;  // an empty range still publishes its totals / finalises
    k_compact_onepass<<<(unsigned)nblk, kCompactThreads, 0, L.stream>>>(a);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// A3 gather + commit.  Units [u_lo, u_hi) of the range whose running totals
// are rb[0] (before) and rb[1] (after); dst == nullptr: commit only;
// no_commit: copy only (a host gather into an image smaller than the worst
// case commits after the whole image is known to fit).
// Unit u is written at dst + (add_poff ? st->poff : 0) + (u - dst_unit0) * 4096.
// ---------------------------------------------------------------------------
constexpr uint32_t kUnitsPerTask = 8;

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

// Largest k in [lo, hi) with sunit[k] <= u.
__device__ __forceinline__ uint64_t slot_of_unit(const uint64_t *sunit, uint64_t lo, uint64_t hi, uint64_t u) {
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (sunit[mid] <= u) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_gather(GatherArgs a) {
    const DevStats *st = a.st;
    if (st->status != kStOk) return;
    const uint64_t k_lo = a.rb[0].k, k_hi = a.rb[1].k;
    const uint64_t u_lo = max(a.u_lo, a.rb[0].units), u_hi = min(a.u_hi, a.rb[1].units);
    if (u_hi <= u_lo) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    uint8_t *payload = a.dst ? a.dst + (a.add_poff ? st->poff : 0) : nullptr;
    // units per task: up to kUnitsPerTask (one slot search per task), fewer
    // when the dirty set is small so every warp gets work
    const uint64_t upt = max((uint64_t)1, min((uint64_t)kUnitsPerTask, (u_hi - u_lo + nwarps - 1) / nwarps));
    const uint64_t ntask = (u_hi - u_lo + upt - 1) / upt;
    for (uint64_t t = (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5); t < ntask; t += nwarps) {
        const uint64_t u0 = u_lo + t * upt, u1 = min(u0 + upt, u_hi);
        uint64_t k = a.u2s[u0];  // slot of the task's first unit (compaction's map)
        uint64_t gid = a.gids[k];
        uint32_t r = region_of_page(a.regs, a.R, gid);
        DevRegion g = a.regs[r];
        uint64_t kbase = a.sunit[k];
        for (uint64_t u = u0; u < u1; ++u) {
            const uint64_t nxt = (k + 1 < k_hi) ? a.sunit[k + 1] : ~0ull;
            if (u >= nxt) {
                ++k;
                kbase = nxt;
                gid = a.gids[k];
                if (r + 1 < a.R && gid >= a.regs[r + 1].page_base) {
                    r = region_of_page(a.regs, a.R, gid);
                    g = a.regs[r];
                }
            }
            const uint64_t seg = u - kbase;
            const uint64_t i = gid - g.page_base;
            const uint64_t off = (i << g.log2p) + (seg << kSegLog2);
            const uint64_t len = g.bytes > off ? min((uint64_t)kSegBytes, g.bytes - off) : 0;
            uint8_t *dst_img = payload ? payload + ((u - a.dst_unit0) << kSegLog2) : nullptr;
            uint8_t *dst_mir = (g.mode == kModeCompare && !a.no_commit) ? g.mirror + off : nullptr;
            if (dst_img || dst_mir) copy_unit(g.base + off, len, g.aligned32 != 0, dst_img, dst_mir, lane);
            if (seg == 0 && lane == 0 && !a.no_commit) {
                if (g.mode == kModeHash) g.table[i] = a.newhash[gid];
                a.force[gid] = 0;
            }
        }
    }
}

void launch_gather(const Launch &L, const GatherArgs &a, uint64_t max_units) {
    if (!a.R || !max_units) return;
    uint64_t blocks = (max_units + kUnitsPerTask * 8 - 1) / (kUnitsPerTask * 8);
    const uint64_t cap = (uint64_t)L.sms * 8;
    if (blocks > cap) blocks = cap;
    if (!blocks) blocks = 1;
    k_gather<<<(unsigned)blocks, 256, 0, L.stream>>>(a);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// CRC-32 (zlib) of table || ids || hashes, copy of the tail into the image,
// header (last block).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t gf2_mulmod(uint32_t a, uint32_t b) {
    // reflected GF(2)[x] product mod the CRC-32 polynomial (the loop ends at
    // the lowest set bit of a, so a == 0 is handled up front)
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

// The same product in a fixed 32 steps without branches: for operands that
// differ across the lanes of a warp, where the early exit above diverges.
__device__ __forceinline__ uint32_t gf2_mulmod_bf(uint32_t a, uint32_t b) {
    uint32_t p = 0;
#pragma unroll
    for (int i = 31; i >= 0; --i) {
        p ^= b & (0u - ((a >> i) & 1u));
        b = (b >> 1) ^ (0xEDB88320u & (0u - (b & 1u)));
    }
    return p;
}

// Raw CRC registers of 16-byte chunks counted from the END of a word stream
// (chunk q is followed by 16 q bytes, so it is placed by x^(128 q)).  Thread
// t of n takes chunks t, t + n, ... and folds them by Horner with
// rpw = x^(128 n); the result still needs x^(128 t).  The (possibly short)
// chunk holding word 0 carries zlib's ~0 initial register.
template <class WordFn>
__device__ __forceinline__ uint32_t crc_chunks_from_end(const WordFn &word, uint64_t nw, uint32_t t, uint32_t n,
                                                        uint32_t rpw, const uint32_t *T) {
    const uint64_t nchunks = (nw + 3) / 4;
    uint32_t acc = 0;
    for (uint64_t r = (nchunks + n - 1) / n; r-- > 0;) {
        if (acc) acc = gf2_mulmod_bf(rpw, acc);
        const uint64_t q = r * n + t;
        if (q < nchunks) {
            const uint64_t wend = nw - 4 * q, wbeg = wend > 4 ? wend - 4 : 0;
            uint32_t c = wbeg == 0 ? 0xffffffffu : 0u;
            for (uint64_t w = wbeg; w < wend; ++w) {
                const uint32_t v = word(w);
#pragma unroll
                for (int b = 0; b < 4; ++b) c = T[(c ^ (v >> (8 * b))) & 0xffu] ^ (c >> 8);
            }
            acc ^= c;
        }
    }
    return acc;
}

__device__ __forceinline__ void put32(uint8_t *p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
__device__ __forceinline__ void put64(uint8_t *p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

// The metadata stream is a whole number of u32 words (48R + round_up(4K,8) +
// 8K bytes).  It is cut into 64-byte chunks counted from the END, so chunk i
// is followed by exactly 64*i bytes: its raw CRC is placed by a product with
// x^(512 i).  A warp takes 32 consecutive chunks (a "task"): lane j shifts by
// pw[j] = x^(512 j), the warp XOR-reduces, and task t is shifted once more by
// x^(8 * 2048 t).  The (possibly short) chunk holding byte 0 carries zlib's
// ~0 initial register.
constexpr uint32_t kCrcWords = 16;

// Slicing-by-4 tables: T[k][n] = CRC register after byte n followed by k
// zero bytes, so one 32-bit word costs 4 independent lookups instead of 4
// dependent ones.
struct CrcSmem {
    uint32_t T[4][256];
    uint32_t x2n[32];
    uint32_t pw[32];
};

__device__ __forceinline__ uint32_t crc_word4(const CrcSmem &sm, uint32_t c) {
    return sm.T[3][c & 0xffu] ^ sm.T[2][(c >> 8) & 0xffu] ^ sm.T[1][(c >> 16) & 0xffu] ^ sm.T[0][c >> 24];
}

__device__ __forceinline__ void crc_smem_init(CrcSmem &sm, const X2N &x) {
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) {
        const uint32_t k = i >> 8;
        uint32_t c = i & 0xffu;
        for (uint32_t b = 0; b < 8 * (k + 1); ++b) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
        sm.T[k][i & 0xffu] = c;
    }
    if (threadIdx.x < 32) {
        sm.x2n[threadIdx.x] = x.t[threadIdx.x];
        sm.pw[threadIdx.x] = x.pw[threadIdx.x];
    }
    __syncthreads();
}

// XOR of the placed CRC terms of this warp's tasks (valid in every lane).
template <class WordFn>
__device__ __forceinline__ uint32_t crc_stream_terms(const WordFn &word, uint64_t nwords, const CrcSmem &sm) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nchunks = (nwords + kCrcWords - 1) / kCrcWords;
    const uint64_t ntasks = (nchunks + 31) / 32;
    uint32_t acc = 0;
    for (uint64_t t = gw; t < ntasks; t += nwarps) {
        const uint64_t i = t * 32 + lane;
        uint32_t raw = 0;
        if (i < nchunks) {
            const uint64_t wend = nwords - i * kCrcWords;
            const uint64_t wbeg = wend > kCrcWords ? wend - kCrcWords : 0;
            const uint32_t n = (uint32_t)(wend - wbeg);
            uint32_t v[kCrcWords];
#pragma unroll
            for (int j = 0; j < (int)kCrcWords; ++j) v[j] = (uint32_t)j < n ? word(wbeg + j) : 0u;
            raw = (wbeg == 0) ? 0xffffffffu : 0u;
#pragma unroll
            for (int j = 0; j < (int)kCrcWords; ++j) {
                if ((uint32_t)j < n) raw = crc_word4(sm, raw ^ v[j]);
            }
        }
        uint32_t term = gf2_mulmod(sm.pw[lane], raw);  // first operand is never 0
#pragma unroll
        for (int o = 16; o; o >>= 1) term ^= __shfl_xor_sync(0xffffffffu, term, o);
        if (t) term = gf2_mulmod(xpow8n(t * 32 * kCrcWords * 4, sm.x2n), term);
        acc ^= term;
    }
    return acc;
}

__global__ void __launch_bounds__(256) k_crc_meta(CrcArgs a) {
    DevStats *st = a.st;
    if (st->status != kStOk) {  // CAPACITY: nothing is written; the stats still reach the host
        if (blockIdx.x == 0 && threadIdx.x == 0 && a.st_host) {
            const uint64_t *src = reinterpret_cast<const uint64_t *>(st);
            volatile uint64_t *dst = reinterpret_cast<volatile uint64_t *>(a.st_host);
            for (uint32_t i = 0; i < sizeof(DevStats) / 8; ++i) dst[i] = src[i];
        }
        return;
    }
    __shared__ CrcSmem sm;
    __shared__ bool s_last;
    crc_smem_init(sm, a.x2n);
    const uint64_t K = st->K, R = st->n_regions;
    const bool hh = (st->img_flags & 2u) != 0;
    const bool zz = (st->img_flags & 4u) != 0;  // compressed: + the u16 unit sizes
    const uint64_t U = st->total_units;
    const uint64_t zw = zz ? round_up(2 * U, 8) / 4 : 0;
    const uint64_t tabw = 12 * R, idsw = round_up(4 * K, 8) / 4, hw = hh ? 2 * K : 0;
    const uint64_t nwords = tabw + idsw + hw + zw;
    uint8_t *tail = a.tail ? a.tail : (a.out ? a.out : a.head) + st->ids_off;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    if (a.out) {  // table + padding into the mapped image (64 + 48 R and poff are multiples of 16)
        const uint4 *src = reinterpret_cast<const uint4 *>(a.head + 64);
        uint4 *dst = reinterpret_cast<uint4 *>(a.out + 64);
        for (uint64_t q = tid; q < (st->poff - 64) / 16; q += nth) dst[q] = src[q];
    }
    // copy ids (+pad) and hashes into the image tail
    uint32_t *tids = reinterpret_cast<uint32_t *>(tail);
    for (uint64_t k = tid; k < idsw; k += nth) tids[k] = k < K ? a.lids[k] : 0u;
    if (hh) {
        uint64_t *th = reinterpret_cast<uint64_t *>(tail + 4 * idsw);
        for (uint64_t k = tid; k < K; k += nth) th[k] = a.lhash[k];
    }
    const uint16_t *zsz = a.zsz;
    if (zz) {
        uint16_t *tz = reinterpret_cast<uint16_t *>(tail + 4 * (idsw + hw));
        for (uint64_t q = tid; q < 2 * zw; q += nth) tz[q] = q < U ? zsz[q] : (uint16_t)0;
    }
    // runs of consecutive page ids (a run starts at a region's page 0 or after a gap)
    uint64_t runs = 0;
    for (uint64_t k = tid; k < K; k += nth)
        runs += (k == 0 || a.lids[k] == 0 || a.gids[k - 1] + 1 != a.gids[k]) ? 1 : 0;
    runs = warp_sum(runs);
    if ((threadIdx.x & 31) == 0 && runs)
        atomicAdd(reinterpret_cast<unsigned long long *>(&st->dirty_runs), (unsigned long long)runs);
    // CRC of table || ids(padded) || hashes, read from the table and the scratch
    const uint32_t *tabp = reinterpret_cast<const uint32_t *>(a.head + 64);
    const uint32_t *lids = a.lids;
    const uint64_t *lhash = a.lhash;
    auto word = [&](uint64_t w) -> uint32_t {
        if (w < tabw) return tabp[w];
        w -= tabw;
        if (w < idsw) return w < K ? lids[w] : 0u;
        w -= idsw;
        if (w < hw) return (uint32_t)(lhash[w >> 1] >> (32 * (w & 1)));
        w -= hw;
        const uint64_t q = 2 * w;
        return (q < U ? (uint32_t)zsz[q] : 0u) | ((q + 1 < U ? (uint32_t)zsz[q + 1] : 0u) << 16);
    };
    const uint32_t acc = crc_stream_terms(word, nwords, sm);
    uint32_t total;
    if (gridDim.x == 1) {
        // one block: XOR the warps' terms in shared memory (no atomics, fence
        // or last-block election)
        __shared__ uint32_t s_acc[32];
        if ((threadIdx.x & 31) == 0) s_acc[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x != 0) return;
        total = st->crc_acc;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) total ^= s_acc[w];
        st->crc_acc = total;
    } else {
        if ((threadIdx.x & 31) == 0 && acc) atomicXor(&st->crc_acc, acc);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = (atomicAdd(a.done, 1u) == gridDim.x - 1);
        __syncthreads();
        if (!s_last || threadIdx.x != 0) return;
        __threadfence();
        *a.done = 0;
        total = *(volatile uint32_t *)&st->crc_acc;
    }
    // empty stream: zlib crc32("") == 0
    const uint32_t meta_crc = (nwords == 0) ? 0u : (total ^ 0xffffffffu);
    st->meta_crc = meta_crc;
    alignas(16) uint8_t h[64];
    h[0] = 'C'; h[1] = 'R'; h[2] = 'U'; h[3] = 'M';
    put32(h + 4, 1);
    put32(h + 8, st->img_flags);
    put32(h + 12, (uint32_t)R);
    put64(h + 16, K);
    put64(h + 24, st->poff);
    put64(h + 32, st->payload_bytes);
    put64(h + 40, st->ids_off);
    put64(h + 48, st->image_bytes);
    put32(h + 56, meta_crc);
    uint32_t c = 0xffffffffu;
    for (int i = 0; i < 60; i += 4)
        c = crc_word4(sm, c ^ ((uint32_t)h[i] | (uint32_t)h[i + 1] << 8 | (uint32_t)h[i + 2] << 16 |
                               (uint32_t)h[i + 3] << 24));
    put32(h + 60, c ^ 0xffffffffu);
    for (int i = 0; i < 64; ++i) a.head[i] = h[i];
    if (a.out)
        for (int i = 0; i < 64; i += 16) *reinterpret_cast<uint4 *>(a.out + i) = *reinterpret_cast<const uint4 *>(h + i);
    if (a.st_host) {
        const uint64_t *src = reinterpret_cast<const uint64_t *>(st);
        volatile uint64_t *dst = reinterpret_cast<volatile uint64_t *>(a.st_host);
        for (uint32_t i = 0; i < sizeof(DevStats) / 8; ++i) dst[i] = src[i];
    }
}

void launch_crc_meta(const Launch &L, const CrcArgs &a, uint64_t max_len) {
    uint64_t blocks = (max_len / (kCrcWords * 4 * 32) + 7) / 8;  // 8 warps per block, 1 task each
    if (blocks < 1) blocks = 1;
    if (blocks > (uint64_t)L.sms * 2) blocks = L.sms * 2;
    k_crc_meta<<<(unsigned)blocks, 256, 0, L.stream>>>(a);
    ++*L.counter;
}

// CRC terms only (restore validation): table || tail into st->crc_acc (the
// host finalises).  Both lengths are multiples of 4.
__global__ void __launch_bounds__(256) k_crc_check(const uint32_t *__restrict__ table, uint64_t tabw,
                                                   const uint32_t *__restrict__ tail, uint64_t tailw, DevStats *st,
                                                   X2N x2n) {
    __shared__ CrcSmem sm;
    crc_smem_init(sm, x2n);
    auto word = [&](uint64_t w) -> uint32_t { return w < tabw ? table[w] : tail[w - tabw]; };
    const uint32_t acc = crc_stream_terms(word, tabw + tailw, sm);
    if ((threadIdx.x & 31) == 0 && acc) atomicXor(&st->crc_acc, acc);
}

void launch_crc_check(const Launch &L, const uint8_t *table, uint64_t tab, const uint8_t *tail, uint64_t tl,
                      DevStats *st, const X2N &x2n) {
    uint64_t blocks = ((tab + tl) / (kCrcWords * 4 * 32) + 7) / 8;
    if (blocks < 1) blocks = 1;
    if (blocks > (uint64_t)L.sms * 2) blocks = L.sms * 2;
    k_crc_check<<<(unsigned)blocks, 256, 0, L.stream>>>(reinterpret_cast<const uint32_t *>(table), tab / 4,
                                                        reinterpret_cast<const uint32_t *>(tail), tl / 4, st, x2n);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// A6 restore: validation of the id list, then scatter + commit.
// rs[] comes from the image's region table (validated on the host); tregs
// are descriptors built from that table (n_pages, mode, page size).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t region_of_slot(const RegStat *rs, uint32_t R, uint64_t k) {
    // the LAST region whose first slot is <= k (regions listing no slot share
    // `first` with their successor)
    uint32_t lo = 0, hi = R;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (rs[mid].first <= k) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_restore_validate(const DevRegion *__restrict__ tregs, uint32_t R,
                                                          const RegStat *__restrict__ rs,
                                                          const uint32_t *__restrict__ ids,
                                                          const uint64_t *__restrict__ hashes, uint64_t K,
                                                          DevStats *st) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    uint32_t bad = 0;
    uint64_t dbytes = 0, runs = 0;
    for (uint64_t k = tid; k < K; k += nth) {
        const uint32_t r = region_of_slot(rs, R, k);
        const DevRegion g = tregs[r];
        const uint64_t i = ids[k];
        const bool first = (k == rs[r].first);
        if (i >= g.n_pages) bad = 1;
        if (!first && ids[k - 1] >= i) bad = 1;
        if (hashes && g.mode != kModeHash && hashes[k] != 0) bad = 1;
        if (i < g.n_pages) dbytes += page_len(g, i);
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

void launch_restore_validate(const Launch &L, const DevRegion *tregs, uint32_t R, const RegStat *rs,
                             const uint32_t *ids, const uint64_t *hashes, uint64_t K, DevStats *st) {
    if (!R || !K) return;
    k_restore_validate<<<L.sms * 2, 256, 0, L.stream>>>(tregs, R, rs, ids, hashes, K, st);
    ++*L.counter;
}

__device__ __forceinline__ uint32_t region_of_unit(const RegStat *rs, uint32_t R, uint64_t u) {
    uint32_t lo = 0, hi = R;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (rs[mid].unit_base <= u) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_scatter(ScatterArgs a) {
    if (a.st->status != kStOk) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nwarps = (uint64_t)gridDim.x * wpb;
    for (uint64_t u = a.u_lo + (uint64_t)blockIdx.x * wpb + (threadIdx.x >> 5); u < a.u_hi; u += nwarps) {
        const uint32_t r = region_of_unit(a.rs, a.R, u);
        const DevRegion g = a.regs[r];
        const RegStat s = a.rs[r];
        const uint32_t sh = g.log2p - kSegLog2;
        const uint64_t ru = u - s.unit_base;
        const uint64_t j = ru >> sh, seg = ru & ((1ull << sh) - 1);
        const uint64_t k = s.first + j;
        if (a.skip && a.skip[k]) continue;
        const uint64_t i = a.ids[k];
        const uint64_t off = (i << g.log2p) + (seg << kSegLog2);
        if (g.bytes > off) {
            const uint64_t len = min((uint64_t)kSegBytes, g.bytes - off);
            const uint8_t *src = a.src + ((u - a.src_unit0) << kSegLog2);
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
            if (g.mode == kModeHash) g.table[i] = a.hashes[k];
            a.force[g.page_base + i] = 0;
            if (a.mark) a.mark[k] = 1;
        }
    }
}

void launch_scatter(const Launch &L, const ScatterArgs &a) {
    if (a.u_hi <= a.u_lo || !a.R) return;
    uint64_t blocks = (a.u_hi - a.u_lo + 7) / 8;
    const uint64_t cap = (uint64_t)L.sms * 8;
    if (blocks > cap) blocks = cap;
    k_scatter<<<(unsigned)blocks, 256, 0, L.stream>>>(a);
    ++*L.counter;
}

// ---------------------------------------------------------------------------
// debug: (flags == tag) | force, global page order
// ---------------------------------------------------------------------------
// crum_mark_dirty_pages: force[pages[k]] = 1 for in-range indices.
__global__ void k_mark_pages(uint8_t *force, uint64_t n_pages, const uint32_t *pages, uint64_t n) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = pages[k];
        if (i < n_pages) force[i] = 1;
    }
}

void launch_mark_pages(const Launch &L, uint8_t *force, uint64_t n_pages, const uint32_t *pages, uint64_t n) {
    if (!n) return;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > (uint64_t)L.sms * 8) blocks = L.sms * 8;
    k_mark_pages<<<(unsigned)blocks, 256, 0, L.stream>>>(force, n_pages, pages, n);
    ++*L.counter;
}

__global__ void k_export_flags(uint8_t *flags, const uint8_t *force, uint64_t N, uint8_t tag, uint8_t *out) {
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < N;
         g += (uint64_t)gridDim.x * blockDim.x) {
        out[g] = (flags[g] == tag || force[g]) ? 1 : 0;
        flags[g] = 0;  // consumed (as by compaction)
    }
}

void launch_export_flags(const Launch &L, uint8_t *flags, const uint8_t *force, uint64_t N, uint8_t tag,
                         uint8_t *out) {
    if (!N) return;
    k_export_flags<<<L.sms * 4, 256, 0, L.stream>>>(flags, force, N, tag, out);
    ++*L.counter;
}

// ===========================================================================
// Single-pass checkpoint for contexts whose regions are all COMPARE mode with
// pages <= 64 KiB (SURVEY.md sec. 7.3 hard part 1): one persistent kernel does
// A1 detect, A2 compaction and A3 gather + commit.
//
//  * Work unit: a tile of max(P, 32 KiB) bytes of one region, claimed through
//    a ticket counter (so every predecessor of a tile is held by a running
//    CTA: the look-back below cannot deadlock).
//  * Detect: 8 warps compare 4 KiB segments (LDG.256, as k_detect_compare)
//    and mark the tile's dirty pages in shared memory.
//  * Compaction: the tile publishes its (dirty pages, 4 KiB units) aggregate,
//    then warp 0 looks back over predecessor status words 32 at a time
//    (decoupled look-back) until it meets an inclusive prefix; the tile's
//    slot and payload offsets follow.  Deterministic: offsets come from
//    prefix sums only, so the image is canonical.
//  * Gather + commit: the dirty pages (just read, so L2-resident) are copied
//    to the image payload and the mirror; slot metadata (ids) is written for
//    the CRC kernel; force bits cleared.
//  * The last CTA to finish a tile finalises (region table, header fields).
// Status word: [63:56] tag, [55:54] state (1 aggregate, 2 inclusive prefix),
// [53:27] dirty pages, [26:0] units (so footprints < 512 GiB).
// ===========================================================================
constexpr uint32_t kFusedThreads = 128;
constexpr uint64_t kStAgg = 1, kStPrefix = 2;

__device__ __forceinline__ uint64_t pack_status(uint32_t tag, uint64_t state, uint64_t cnt, uint64_t units) {
    return ((uint64_t)tag << 56) | (state << 54) | ((cnt & 0x7ffffffull) << 27) | (units & 0x7ffffffull);
}
__device__ __forceinline__ void st_release(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// A look-back status word is self-contained (tag, state, count, units in one
// 64-bit word) and nothing else a predecessor wrote is read on the strength
// of it (the finalising warp synchronises through the done counter), so
// relaxed GPU-scope accesses suffice: no fence per load / store.
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void ld256(const void *p, uint32_t (&r)[8]) {
    asm volatile("ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "l"(p));
}

// Warp-exclusive scan of u64 (returns exclusive prefix, *total = warp sum).
__device__ __forceinline__ uint64_t warp_excl_scan(uint64_t v, uint64_t *total) {
    const uint32_t lane = threadIdx.x & 31;
    uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += t;
    }
    *total = __shfl_sync(0xffffffffu, inc, 31);
    return inc - v;
}

// Small footprints: the finalising warp also does k_crc_meta's work for
// this image -- ids (+ pad) into the tail, runs, the zlib CRC-32 of table ||
// ids (32 lane chunks, each a raw register shifted into place by
// x^(8 * bytes after it)), and the header with its own CRC -- so the whole
// checkpoint is one kernel.  Compare-only contexts: no hashes, no sizes.
__device__ __noinline__ void fused_inline_meta(const FusedArgs &a, uint64_t K, uint64_t U, uint64_t poff,
                                               uint32_t lane) {
    __shared__ uint32_t T[256];  // byte-wise CRC-32 table (reflected polynomial)
    for (uint32_t i = lane; i < 256; i += 32) {
        uint32_t c = i;
        for (int b = 0; b < 8; ++b) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
        T[i] = c;
    }
    DevStats *st = a.st;
    const uint64_t payload = U << kSegLog2, ids_off = poff + payload;
    const uint64_t idsw = round_up(4 * K, 8) / 4;
    uint32_t *tids = reinterpret_cast<uint32_t *>(a.img + ids_off);
    for (uint64_t k = lane; k < idsw; k += 32) tids[k] = k < K ? a.lids[k] : 0u;
    uint64_t runs = 0;
    for (uint64_t k = lane; k < K; k += 32) runs += (k == 0 || a.lids[k] == 0 || a.gids[k - 1] + 1 != a.gids[k]) ? 1 : 0;
    runs = warp_sum(runs);
    __syncwarp();
    // CRC of table (12 R words at img + 64) || ids (idsw words, from lids):
    // 16-byte chunks from the end, lane j's placed by x^(128 j)
    const uint64_t tabw = 12ull * a.R, nw = tabw + idsw;
    const uint32_t *tab = reinterpret_cast<const uint32_t *>(a.img + 64);
    auto word = [&](uint64_t w) -> uint32_t {
        return w < tabw ? tab[w] : ((w - tabw) < K ? a.lids[w - tabw] : 0u);
    };
    uint32_t term = crc_chunks_from_end(word, nw, lane, 32, a.x2n.t[12], T);
    term = gf2_mulmod_bf(a.x2n.lpw[lane], term);
#pragma unroll
    for (int o = 16; o; o >>= 1) term ^= __shfl_xor_sync(0xffffffffu, term, o);
    if (lane != 0) return;
    st->dirty_runs = runs;
    const uint32_t meta_crc = nw == 0 ? 0u : (term ^ 0xffffffffu);
    st->meta_crc = meta_crc;
    uint8_t h[64];
    h[0] = 'C'; h[1] = 'R'; h[2] = 'U'; h[3] = 'M';
    put32(h + 4, 1);
    put32(h + 8, 0);  // incremental, no hashes, not compressed
    put32(h + 12, a.R);
    put64(h + 16, K);
    put64(h + 24, poff);
    put64(h + 32, payload);
    put64(h + 40, ids_off);
    put64(h + 48, ids_off + 4 * idsw);
    put32(h + 56, meta_crc);
    uint32_t hc = 0xffffffffu;
    for (int i = 0; i < 60; ++i) hc = T[(hc ^ h[i]) & 0xffu] ^ (hc >> 8);
    put32(h + 60, hc ^ 0xffffffffu);
    for (int i = 0; i < 64; ++i) a.img[i] = h[i];
    if (a.st_host) {  // the host reads the report without a copy
        const uint64_t *src = reinterpret_cast<const uint64_t *>(st);
        volatile uint64_t *dst = reinterpret_cast<volatile uint64_t *>(a.st_host);
        for (uint32_t i = 0; i < sizeof(DevStats) / 8; ++i) dst[i] = src[i];
    }
}

// Each WARP owns one tile at a time: no block barriers, so while one warp
// waits in its look-back the SM's other warps keep streaming.
__global__ void __launch_bounds__(kFusedThreads) k_fused_compare(FusedArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    bool last = false;
    for (;;) {
        uint64_t t = 0;
        if (lane == 0) t = atomicAdd(&a.fs->ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= a.n_tiles) break;
        // tile -> region, byte range
        uint32_t r;
        {
            uint32_t lo = 0, hi = a.R;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(a.tile_base + mid) <= t) lo = mid; else hi = mid;
            }
            r = lo;
        }
        const DevRegion g = a.regs[r];
        const uint32_t tlog = max(g.log2p, a.tile_log2_min);
        const uint64_t off0 = (t - __ldg(a.tile_base + r)) << tlog;
        const uint64_t tlen = min((uint64_t)1 << tlog, g.bytes - off0);
        const uint64_t i0 = off0 >> g.log2p;  // first page of the tile
        const uint32_t npg = (uint32_t)((tlen + (1ull << g.log2p) - 1) >> g.log2p);
        const uint32_t nseg = (uint32_t)((tlen + kSegBytes - 1) >> kSegLog2);
        const uint32_t spl = g.log2p - kSegLog2;  // log2 segments per page
        // ---- A1 detect: force bits, then 4 KiB segments; a page found dirty
        // stops being compared (its bytes are gathered below anyway) ----
        uint32_t dmask = __ballot_sync(0xffffffffu, lane < npg && a.force[g.page_base + i0 + lane] != 0);
        for (uint32_t sg = 0; sg < nseg; ++sg) {
            const uint32_t j = sg >> spl;
            if ((dmask >> j) & 1u) continue;
            const uint64_t off = off0 + ((uint64_t)sg << kSegLog2);
            const uint64_t len = g.bytes - off;
            const uint8_t *pa = g.base + off, *pb = g.mirror + off;
            // the next segment's lines into L2 while this one is compared: a
            // warp walks its tile serially, so one segment of loads in flight
            // per warp (plus the prefetch) instead of one
            if (a.prefetch && sg + 1 < nseg && len >= 2 * kSegBytes) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + kSegBytes + lane * 128));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + kSegBytes + lane * 128));
            }
            uint32_t x = 0;
            if (len >= kSegBytes && g.aligned32) {
                uint32_t va[4][8], vb[4][8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    ld256(pa + i * 1024 + lane * 32, va[i]);
                    ld256(pb + i * 1024 + lane * 32, vb[i]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int k = 0; k < 8; ++k) x |= va[i][k] ^ vb[i][k];
            } else if (len >= kSegBytes) {
                for (int i = 0; i < 8; ++i) {
                    const uint4 u = *reinterpret_cast<const uint4 *>(pa + i * 512 + lane * 16);
                    const uint4 v = *reinterpret_cast<const uint4 *>(pb + i * 512 + lane * 16);
                    x |= (u.x ^ v.x) | (u.y ^ v.y) | (u.z ^ v.z) | (u.w ^ v.w);
                }
            } else {
                for (uint32_t o = lane; o < len; o += 32) x |= (uint32_t)(pa[o] ^ pb[o]);
            }
            if (__any_sync(0xffffffffu, x != 0)) dmask |= 1u << j;
        }
        // ---- A2 compaction: aggregate, look-back, inclusive prefix ----
        const uint32_t cnt = __popc(dmask);
        const uint64_t ucnt = (uint64_t)cnt << spl;
        if (lane == 0) st_relaxed(a.status + t, pack_status(a.tag, kStAgg, cnt, ucnt));
        // look back kLB windows of 32 predecessors per step: the status loads
        // of a step are independent, so a step costs one round trip however
        // far the nearest inclusive prefix is (small footprints: when every
        // tile starts at once, prefixes are rare and one-window steps made the
        // last tiles wait ~n/32 round trips)
        constexpr int kLB = 8;
        uint64_t ec = 0, eu = 0;
        int64_t top = (int64_t)t - 1;
        while (top >= 0) {
            uint64_t v[kLB];
            uint32_t stt[kLB];
#pragma unroll
            for (int j = 0; j < kLB; ++j) {
                const int64_t idx = top - (int64_t)lane - 32 * j;
                v[j] = pack_status(a.tag, kStPrefix, 0, 0);  // before tile 0: prefix 0
                stt[j] = (uint32_t)kStPrefix;
                if (idx >= 0) {
                    v[j] = ld_relaxed(a.status + idx);
                    stt[j] = ((v[j] >> 56) == a.tag) ? (uint32_t)((v[j] >> 54) & 3) : 0u;
                }
            }
#pragma unroll
            for (int j = 0; j < kLB; ++j) {  // wait for the ones not yet published
                const int64_t idx = top - (int64_t)lane - 32 * j;
                while (stt[j] == 0) {
                    v[j] = ld_relaxed(a.status + idx);
                    stt[j] = ((v[j] >> 56) == a.tag) ? (uint32_t)((v[j] >> 54) & 3) : 0u;
                }
            }
            // nearest inclusive prefix: smallest distance 32 j + lane
            uint32_t mine = 0xffffffffu;
#pragma unroll
            for (int j = kLB - 1; j >= 0; --j)
                if (stt[j] == kStPrefix) mine = 32 * j + lane;
            const uint32_t first = __reduce_min_sync(0xffffffffu, mine);
            uint64_t c = 0, u = 0;
#pragma unroll
            for (int j = 0; j < kLB; ++j)
                if (32u * j + lane <= first) {
                    c += (v[j] >> 27) & 0x7ffffffull;
                    u += v[j] & 0x7ffffffull;
                }
            ec += warp_sum(c);
            eu += warp_sum(u);
            if (first != 0xffffffffu) break;
            top -= 32 * kLB;
        }
        if (lane == 0) st_relaxed(a.status + t, pack_status(a.tag, kStPrefix, ec + cnt, eu + ucnt));
        // ---- A3 gather + commit: the tile's dirty pages, ascending ----
        uint32_t m = dmask;
        for (uint32_t rank = 0; m; ++rank, m &= m - 1) {
            const uint32_t j = __ffs(m) - 1;
            const uint64_t i = i0 + j;
            const uint64_t pg_off = i << g.log2p;
            const uint64_t dst_u = eu + ((uint64_t)rank << spl);
            for (uint32_t sg = 0; sg < (1u << spl); ++sg) {
                const uint64_t off = pg_off + ((uint64_t)sg << kSegLog2);
                const uint64_t len = g.bytes > off ? min((uint64_t)kSegBytes, g.bytes - off) : 0;
                copy_unit(g.base + off, len, g.aligned32 != 0, a.img + a.poff + ((dst_u + sg) << kSegLog2),
                          g.mirror + off, lane);
            }
        }
        uint64_t db = 0;
        if (lane < 32 && ((dmask >> lane) & 1u)) {
            const uint32_t rank = __popc(dmask & ((1u << lane) - 1));
            const uint64_t i = i0 + lane;
            const uint64_t k = ec + rank;
            a.gids[k] = (uint32_t)(g.page_base + i);
            a.sunit[k] = eu + ((uint64_t)rank << spl);
            a.lids[k] = (uint32_t)i;
            a.force[g.page_base + i] = 0;
            db = page_len(g, i);
        }
        db = warp_sum(db);
        if (lane == 0 && cnt) {
            atomicAdd(reinterpret_cast<unsigned long long *>(&a.fs->dirty_bytes), (unsigned long long)db);
            atomicAdd(a.reg_nd + r, cnt);
        }
        __threadfence();
        uint32_t f = 0;
        if (lane == 0) f = atomicAdd(&a.fs->done, 1u);
        f = __shfl_sync(0xffffffffu, f, 0);
        if (f == a.n_tiles - 1) {
            last = true;
            break;
        }
    }
    if (!last) return;
    // ---- finalise (the warp that finished the last tile) ----
    __threadfence();
    const uint64_t fin = ld_acquire(a.status + a.n_tiles - 1);
    const uint64_t K = (fin >> 27) & 0x7ffffffull, U = fin & 0x7ffffffull;
    uint64_t carry_first = 0, carry_units = 0;
    for (uint32_t r0 = 0; r0 < a.R; r0 += 32) {
        const uint32_t r = r0 + lane;
        uint64_t nd = 0, un = 0;
        DevRegion g{};
        if (r < a.R) {
            g = a.regs[r];
            nd = *(volatile uint32_t *)(a.reg_nd + r);
            un = nd << (g.log2p - kSegLog2);
        }
        uint64_t tn, tun;
        const uint64_t en = warp_excl_scan(nd, &tn);
        const uint64_t eun = warp_excl_scan(un, &tun);
        if (r < a.R) {
            RegStat s;
            s.first = carry_first + en;
            s.n_dirty = nd;
            s.unit_base = carry_units + eun;
            s.payload_base = s.unit_base << kSegLog2;
            a.rs[r] = s;
            a.reg_nd[r] = 0;  // ready for the next checkpoint
            uint8_t *e = (a.meta ? a.meta : a.img) + 64 + 48ull * r;
            reinterpret_cast<uint32_t *>(e)[0] = g.id;
            reinterpret_cast<uint32_t *>(e)[1] = g.mode;
            reinterpret_cast<uint64_t *>(e)[1] = g.bytes;
            reinterpret_cast<uint64_t *>(e)[2] = 1ull << g.log2p;
            reinterpret_cast<uint64_t *>(e)[3] = g.n_pages;
            reinterpret_cast<uint64_t *>(e)[4] = nd;
            reinterpret_cast<uint64_t *>(e)[5] = s.first;
        }
        carry_first += tn;
        carry_units += tun;
    }
    const uint64_t poff = a.poff;
    for (uint64_t b = 64 + 48ull * a.R + lane; b < poff; b += 32) (a.meta ? a.meta : a.img)[b] = 0;
    if (lane == 0) {
        DevStats *st = a.st;
        const uint64_t payload = U << kSegLog2;
        const uint64_t ids_off = poff + payload;
        st->K = K;
        st->total_units = U;
        st->poff = poff;
        st->payload_bytes = payload;
        st->ids_off = ids_off;
        st->image_bytes = ids_off + round_up(4 * K, 8);
        st->capacity = a.capacity;
        st->status = st->image_bytes > a.capacity ? kStCapacity : kStOk;
        st->img_flags = 0;
        st->n_regions = a.R;
        st->dirty_bytes = a.fs->dirty_bytes;
        st->dirty_runs = 0;
        st->crc_acc = 0;
        // the ticket / done counters are NOT reset here: a warp that is late
        // to its final claim must still see ticket >= n_tiles.  The host
        // zeroes the scratch stream-ordered before every launch.
    }
    __syncwarp();  // the table, padding and stats written by the lanes above
    if (a.inline_meta) fused_inline_meta(a, K, U, poff, lane);
}

// ---------------------------------------------------------------------------
// One-launch small-footprint checkpoint (see SmallArgs).
// ---------------------------------------------------------------------------
constexpr uint32_t kSmallThreads = 256;
constexpr uint32_t kSmallWords = kSmallPages / 32;
constexpr uint32_t kSmallStageWords = 2048;  // metadata words CTA 0 keeps in shared memory

// A GPU-scope acquire-release fence: with the relaxed atomics around it, the
// release / acquire pattern a barrier or a "last one out" election needs --
// lighter than __threadfence() (fence.sc).
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Grid barrier of a cooperative launch (all CTAs co-resident): arrivals
// counter + generation, sense by generation, state returns to 0 arrivals.
// The arrival is one acq_rel atomic (it releases this CTA's bitmap atomics
// and, for the last arrival, acquires everyone's); the last one resets the
// count and publishes the next generation with a release store; the others
// poll an acquire load of the generation, backing off between polls (~500
// CTAs polling one address back to back slowed the release by ~1 us; a
// two-level arrival tree was slower still).
__device__ __forceinline__ void grid_barrier(uint32_t *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t g, old;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(g + 1) : "memory");
        } else {
            uint32_t cur;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
                if (cur != g) break;
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
}

__device__ __forceinline__ uint64_t gtime_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Profiling aid (off in every shipped build): -DCRUM_SMALL_STAMPS records
// globaltimer stamps per CTA and phase (after the barrier words) and the last
// CTA out prints, per phase, the earliest and latest CTA relative to the first
// entry (tools/gpu_r02_c1_stamps.sh).
#ifdef CRUM_SMALL_STAMPS
}  // namespace crum
#include <cstdio>
namespace crum {
constexpr int kStampN = 16;
#define SMALL_STAMP(k)                                                                              \
    do {                                                                                            \
        if (threadIdx.x == 0)                                                                       \
            reinterpret_cast<uint64_t *>(a.bar + 16)[blockIdx.x * kStampN + (k)] = gtime_ns();     \
    } while (0)
__device__ void small_stamps_print(const SmallArgs &a) {
    const uint64_t *t = reinterpret_cast<const uint64_t *>(a.bar + 16);
    uint64_t t0 = ~0ull;
    for (uint32_t b = 0; b < gridDim.x; ++b) t0 = min(t0, t[b * kStampN]);
    for (int k = 0; k < kStampN; ++k) {
        uint64_t lo = ~0ull, hi = 0;
        for (uint32_t b = 0; b < gridDim.x; ++b) {
            const uint64_t v = t[b * kStampN + k];
            if (!v) continue;
            lo = min(lo, v - t0);
            hi = max(hi, v - t0);
        }
        if (hi) printf("[small stamps] phase %d: first %llu ns, last %llu ns\n", k, (unsigned long long)lo,
                       (unsigned long long)hi);
    }
    for (uint32_t i = 0; i < gridDim.x * kStampN; ++i) const_cast<uint64_t *>(t)[i] = 0;
}
#else
#define SMALL_STAMP(k) do {} while (0)
#endif

// Every CTA leaves through here (all threads, after the CTA's work -- which
// includes its last read of the global bitmap).  CTAs 1.. count themselves
// out; CTA 0 (the metadata CTA, the last to finish) waits until they all
// have, then clears the bitmap's nw words for the next launch, publishes the
// stats to the host -- with the kernel's own duration when timed -- and
// returns the scratch words to 0.  CTA 0 itself needs no fence: nobody else
// reads what it wrote during the launch (a fence after its header's stores
// to a pinned image waited ~1.5 us for the host link).  (One bitmap, cleared
// on the way out: a launch needs no generation read before its first load.)
__device__ __forceinline__ void small_leave(const SmallArgs &a, uint32_t nw) {
    __syncthreads();
    SMALL_STAMP(7);
    if (blockIdx.x != 0) {
        if (threadIdx.x == 0) {
            fence_acq_rel_gpu();  // this CTA's bitmap reads and commits before it counts out
            atomicAdd(a.bar + 2, 1u);
        }
        return;
    }
    if (threadIdx.x == 0) {
        uint32_t out;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(out) : "l"(a.bar + 2) : "memory");
        } while (out != gridDim.x - 1);
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < nw; w += blockDim.x) a.bitmap[w] = 0;
    if (threadIdx.x != 0) return;
#ifdef CRUM_SMALL_STAMPS
    small_stamps_print(a);
#endif
    volatile unsigned long long *t0 = reinterpret_cast<volatile unsigned long long *>(a.bar + 4);
    DevStats *st = a.st;
    st->t_ns = a.timing ? gtime_ns() - ~*t0 : 0;
    *t0 = 0;
    a.bar[2] = 0;
    if (a.st_host) {  // the host reads the report without a copy
        const volatile uint64_t *src = reinterpret_cast<const volatile uint64_t *>(st);
        volatile uint64_t *dst = reinterpret_cast<volatile uint64_t *>(a.st_host);
        for (uint32_t i = 0; i < sizeof(DevStats) / 8; ++i) dst[i] = src[i];
    }
}

__global__ void __launch_bounds__(kSmallThreads) k_small_ckpt(SmallArgs a) {
    __shared__ uint32_t s_bm[kSmallWords];    // dirty bitmap
    __shared__ uint32_t s_pre[kSmallWords + 1];  // dirty pages before word w
    __shared__ uint32_t T4[4][256];            // CRC-32 tables (CTA 0): T4[k][i] = byte i then k zero bytes
    uint32_t *T = T4[0];                       // the byte-wise table
    __shared__ uint32_t s_lpw[32];             // x^(128 j) mod P (CTA 0)
    __shared__ uint32_t s_w[kSmallStageWords]; // table || ids words for the CRC (CTA 0)
    const uint32_t lane = threadIdx.x & 31;
    // detect runs on CTAs 1.. (CTA 0, the metadata CTA, builds its CRC tables
    // meanwhile and reaches the barrier early); a one-CTA grid detects itself
    const uint32_t dcta = gridDim.x > 1 ? 1u : 0u;
    const uint64_t wid = ((uint64_t)(blockIdx.x - dcta) * kSmallThreads + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)(gridDim.x - dcta) * kSmallThreads) >> 5;
    const uint32_t spl = a.log2p - kSegLog2;   // log2 segments per page
    const uint64_t P = 1ull << a.log2p;
    if (a.timing && threadIdx.x == 0)  // the max of ~t is the earliest entry
        atomicMax(reinterpret_cast<unsigned long long *>(a.bar + 4), ~(unsigned long long)gtime_ns());
    uint32_t *bitmap = a.bitmap;  // zero when the launch begins (small_leave)
    SMALL_STAMP(0);
    // ---- A1 detect: a warp per 4 KiB >> kSmallItemsLog2 of a segment (more
    // warps than one per 4 KiB: more SMs issue the cold loads at once); a
    // forced page is dirty ----
    constexpr uint32_t kSmallItems = 1u << kSmallItemsLog2;
    uint32_t r = 0;
    for (uint64_t g = wid; blockIdx.x >= dcta && g < (a.N << spl) * kSmallItems; g += nwarps) {
        const uint64_t pg = g >> (spl + kSmallItemsLog2);
        while (r + 1 < a.R && a.regs[r + 1].page_base <= pg) ++r;
        while (a.regs[r].page_base > pg) --r;
        const DevRegion &R = a.regs[r];
        // the force byte is loaded before, and consumed after, the segment's
        // loads (a forced page's compare is wasted, but the loads overlap
        // instead of chaining two cold HBM round trips)
        const uint8_t forced = a.force[pg];
        bool dirty = false;
        if (R.mode == kModeCompare) {
            const uint64_t off = ((pg - R.page_base) << a.log2p) +
                                 ((g & ((kSmallItems << spl) - 1)) << (kSegLog2 - kSmallItemsLog2));
            uint32_t x = 0;
            if (off < R.bytes) {
                const uint64_t len = R.bytes - off;
                const uint8_t *pa = R.base + off, *pb = R.mirror + off;
                if (len >= (kSegBytes >> kSmallItemsLog2)) {
#pragma unroll
                    for (int i = 0; i < (8 >> kSmallItemsLog2); ++i) {
                        const uint4 u = __ldcs(reinterpret_cast<const uint4 *>(pa + i * 512 + lane * 16));
                        const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(pb + i * 512 + lane * 16));
                        x |= (u.x ^ v.x) | (u.y ^ v.y) | (u.z ^ v.z) | (u.w ^ v.w);
                    }
                } else {
                    for (uint32_t o = lane; o < len; o += 32) x |= (uint32_t)(pa[o] ^ pb[o]);
                }
            }
            dirty = __any_sync(0xffffffffu, x != 0);
        }
        dirty = dirty || forced != 0;
        if (dirty && lane == 0) atomicOr(bitmap + (pg >> 5), 1u << (pg & 31));
    }
#ifdef CRUM_SMALL_STAMPS
    __syncthreads();
#endif
    SMALL_STAMP(1);
    if (blockIdx.x == 0) {  // CTA 0's CRC tables, while the barrier waits for the last CTA
        if (threadIdx.x < 32) s_lpw[threadIdx.x] = a.x2n.lpw[threadIdx.x];
        for (uint32_t i = threadIdx.x; i < 256; i += kSmallThreads) {
            uint32_t c = i;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                for (int b = 0; b < 8; ++b) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
                T4[k][i] = c;
            }
        }
    }
    grid_barrier(a.bar);
    SMALL_STAMP(2);
    // ---- A2: every CTA: the bitmap and its word prefix in shared memory ----
    const uint32_t nw = (uint32_t)((a.N + 31) >> 5);
    for (uint32_t w = threadIdx.x; w < nw; w += kSmallThreads) s_bm[w] = __ldcg(bitmap + w);
    __syncthreads();
    {   // exclusive prefix of popc over the words: 256 threads x (nw / 256) words
        const uint32_t per = (nw + kSmallThreads - 1) / kSmallThreads;
        const uint32_t w0 = threadIdx.x * per;
        uint64_t own = 0;
        for (uint32_t w = w0; w < min(nw, w0 + per); ++w) own += __popc(s_bm[w]);
        uint64_t tot;
        uint64_t run = block_excl_scan(own, &tot);
        for (uint32_t w = w0; w < min(nw, w0 + per); ++w) {
            s_pre[w] = (uint32_t)run;
            run += __popc(s_bm[w]);
        }
        if (threadIdx.x == 0) s_pre[nw] = (uint32_t)tot;
    }
    __syncthreads();
    SMALL_STAMP(3);
    const uint64_t K = s_pre[nw];
    // rank k -> page: the word by binary search over s_pre, the bit by select
    auto page_of = [&](uint64_t k) -> uint64_t {
        uint32_t lo = 0, hi = nw;  // largest w with s_pre[w] <= k
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_pre[mid] <= k) lo = mid; else hi = mid;
        }
        uint32_t m = s_bm[lo];
        for (uint32_t j = (uint32_t)(k - s_pre[lo]); j; --j) m &= m - 1;
        return 32ull * lo + (__ffs(m) - 1);
    };
    // ---- A3 gather + commit: warp per dirty page (CTA 0 does the metadata) ----
    const uint64_t gw = blockIdx.x == 0 ? 0 : ((uint64_t)(blockIdx.x - 1) * kSmallThreads + threadIdx.x) >> 5;
    const uint64_t gnw = ((uint64_t)(gridDim.x > 1 ? gridDim.x - 1 : 1) * kSmallThreads) >> 5;
    if (blockIdx.x != 0 || gridDim.x == 1) {
        uint32_t rr = 0;
        for (uint64_t k = (gridDim.x == 1 ? (threadIdx.x >> 5) : gw); k < K; k += (gridDim.x == 1 ? kSmallThreads / 32 : gnw)) {
            const uint64_t pg = page_of(k);
            while (rr + 1 < a.R && a.regs[rr + 1].page_base <= pg) ++rr;
            while (a.regs[rr].page_base > pg) --rr;
            const DevRegion &R = a.regs[rr];
            const uint64_t i = pg - R.page_base;
            uint8_t *dst = a.img + a.poff + (k << a.log2p);
            for (uint32_t sg = 0; sg < (1u << spl); ++sg) {
                const uint64_t off = (i << a.log2p) + ((uint64_t)sg << kSegLog2);
                const uint64_t len = R.bytes > off ? min((uint64_t)kSegBytes, R.bytes - off) : 0;
                uint8_t *d = dst + ((uint64_t)sg << kSegLog2);
                uint8_t *m = R.mode == kModeCompare ? R.mirror + off : nullptr;
                if (len == kSegBytes) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint4 v = *reinterpret_cast<const uint4 *>(R.base + off + j * 512 + lane * 16);
                        *reinterpret_cast<uint4 *>(d + j * 512 + lane * 16) = v;
                        if (m) *reinterpret_cast<uint4 *>(m + j * 512 + lane * 16) = v;
                    }
                } else {
                    for (uint32_t o = lane; o < kSegBytes; o += 32) {
                        const uint8_t v = o < len ? R.base[off + o] : 0;
                        d[o] = v;
                        if (m && o < len) m[o] = v;
                    }
                }
            }
            if (lane == 0) a.force[pg] = 0;
        }
        if (blockIdx.x != 0) {
            small_leave(a, nw);
            return;
        }
    }
    // ---- CTA 0: table, ids, CRC, header ----
    __syncthreads();
    SMALL_STAMP(4);
    SMALL_STAMP(8);
    const uint64_t poff = a.poff, payload = K << a.log2p, ids_off = poff + payload;
    const uint64_t idsw = round_up(4 * K, 8) / 4;
    uint8_t *img = a.img;
    auto prefix_at = [&](uint64_t p) -> uint64_t {  // dirty pages before page p
        const uint32_t w = (uint32_t)(p >> 5), b = (uint32_t)(p & 31);
        return s_pre[w] + (b ? __popc(s_bm[w] & ((1u << b) - 1)) : 0u);
    };
    for (uint32_t rr = threadIdx.x; rr < a.R; rr += kSmallThreads) {
        const DevRegion R = a.regs[rr];
        const uint64_t first = prefix_at(R.page_base), nd = prefix_at(R.page_base + R.n_pages) - first;
        uint8_t *e = img + 64 + 48ull * rr;
        reinterpret_cast<uint32_t *>(e)[0] = R.id;
        reinterpret_cast<uint32_t *>(e)[1] = R.mode;
        reinterpret_cast<uint64_t *>(e)[1] = R.bytes;
        reinterpret_cast<uint64_t *>(e)[2] = P;
        reinterpret_cast<uint64_t *>(e)[3] = R.n_pages;
        reinterpret_cast<uint64_t *>(e)[4] = nd;
        reinterpret_cast<uint64_t *>(e)[5] = first;
        if (12 * rr + 12 <= kSmallStageWords) {
            uint32_t *sw = s_w + 12 * rr;
            sw[0] = R.id;
            sw[1] = R.mode;
            sw[2] = (uint32_t)R.bytes;   sw[3] = (uint32_t)(R.bytes >> 32);
            sw[4] = (uint32_t)P;         sw[5] = (uint32_t)(P >> 32);
            sw[6] = (uint32_t)R.n_pages; sw[7] = (uint32_t)(R.n_pages >> 32);
            sw[8] = (uint32_t)nd;        sw[9] = (uint32_t)(nd >> 32);
            sw[10] = (uint32_t)first;    sw[11] = (uint32_t)(first >> 32);
        }
    }
    // zero padding to the payload: 16-byte stores (64 + 48 R and poff are multiples of 16)
    for (uint64_t b = 64 + 48ull * a.R + 16ull * threadIdx.x; b < poff; b += 16ull * kSmallThreads)
        *reinterpret_cast<uint4 *>(img + b) = make_uint4(0, 0, 0, 0);
    SMALL_STAMP(9);
    // ids (region-local page indices), runs, logical bytes
    uint32_t *tids = reinterpret_cast<uint32_t *>(img + ids_off);
    uint64_t runs = 0, dbytes = 0;
    {
        uint32_t rr = 0;
        for (uint64_t k = threadIdx.x; k < idsw; k += kSmallThreads) {
            if (k >= K) {
                tids[k] = 0;
                if (12ull * a.R + k < kSmallStageWords) s_w[12 * a.R + k] = 0;
                continue;
            }
            const uint64_t pg = page_of(k);
            while (rr + 1 < a.R && a.regs[rr + 1].page_base <= pg) ++rr;
            while (a.regs[rr].page_base > pg) --rr;
            const DevRegion &R = a.regs[rr];
            const uint64_t i = pg - R.page_base;
            tids[k] = (uint32_t)i;
            if (12ull * a.R + k < kSmallStageWords) s_w[12 * a.R + k] = (uint32_t)i;
            runs += (i == 0 || !((s_bm[(pg - 1) >> 5] >> ((pg - 1) & 31)) & 1u)) ? 1 : 0;
            dbytes += min(P, R.bytes - (i << a.log2p));
        }
    }
    SMALL_STAMP(10);
    uint64_t tot_runs, tot_bytes;
    block_excl_scan(runs, &tot_runs);
    block_excl_scan(dbytes, &tot_bytes);
    __syncthreads();  // table, ids and padding written
    SMALL_STAMP(5);
    // CRC-32 of table (12 R words) || ids (idsw words), 16-byte chunks from
    // the end.  The words come from the shared-memory stage, beyond it they
    // are recomputed -- never read back from the image (which may be a pinned
    // image behind the host link).
    const uint64_t tabw = 12ull * a.R, nwords = tabw + idsw;
    uint32_t cr = 0;  // region cursor for the ids
    auto word = [&](uint64_t w) -> uint32_t {
        if (w < kSmallStageWords && (w >= tabw || 12 * (w / 12) + 12 <= kSmallStageWords)) return s_w[w];
        if (w < tabw) {
            const DevRegion &R = a.regs[w / 12];
            uint64_t f = 0;
            switch ((uint32_t)(w % 12) >> 1) {
                case 0: f = ((uint64_t)R.mode << 32) | R.id; break;
                case 1: f = R.bytes; break;
                case 2: f = P; break;
                case 3: f = R.n_pages; break;
                case 4: f = prefix_at(R.page_base + R.n_pages) - prefix_at(R.page_base); break;
                default: f = prefix_at(R.page_base); break;
            }
            return (uint32_t)(f >> (32 * (w & 1)));
        }
        if (w - tabw >= K) return 0u;
        const uint64_t pg = page_of(w - tabw);
        while (cr + 1 < a.R && a.regs[cr + 1].page_base <= pg) ++cr;
        while (a.regs[cr].page_base > pg) --cr;
        return (uint32_t)(pg - a.regs[cr].page_base);
    };
    // thread t = 32 w + lane is placed by x^(128 t) = x^(128 lane) x^(4096 w);
    // a chunk's four words a word per step (slicing by 4: four independent
    // table loads per step instead of a chain of sixteen)
    auto crc_w4 = [&](uint32_t c, uint32_t w) -> uint32_t {
        c ^= w;
        return T4[3][c & 0xffu] ^ T4[2][(c >> 8) & 0xffu] ^ T4[1][(c >> 16) & 0xffu] ^ T4[0][c >> 24];
    };
    uint32_t x = 0;
    {
        const uint64_t nchunks = (nwords + 3) / 4;
        for (uint64_t r = (nchunks + kSmallThreads - 1) / kSmallThreads; r-- > 0;) {
            if (x) x = gf2_mulmod_bf(a.x2n.t[15], x);
            const uint64_t q = r * kSmallThreads + threadIdx.x;
            if (q < nchunks) {
                const uint64_t wend = nwords - 4 * q, wbeg = wend > 4 ? wend - 4 : 0;
                uint32_t c = wbeg == 0 ? 0xffffffffu : 0u;
                for (uint64_t w = wbeg; w < wend; ++w) c = crc_w4(c, word(w));
                x ^= c;
            }
        }
    }
    SMALL_STAMP(11);
    x = gf2_mulmod_bf(s_lpw[lane], x);
#pragma unroll
    for (int o = 16; o; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
    __shared__ uint32_t s_x[kSmallThreads / 32];
    __shared__ uint32_t s_hc;
    if (lane == 0) s_x[threadIdx.x >> 5] = gf2_mulmod_bf(a.x2n.wpw[threadIdx.x >> 5], x);
    // the header's first 56 bytes (14 words, in registers) are known already:
    // their CRC register beside the others, a word per step (slicing by 4)
    const uint64_t iend = ids_off + 4 * idsw;
    const uint32_t hw0 = 0x4D555243u /* "CRUM" */, hw1 = 1u, hw2 = 0u, hw3 = a.R;
    if (threadIdx.x == 32) {
        uint32_t hc = 0xffffffffu;
        hc = crc_w4(hc, hw0); hc = crc_w4(hc, hw1); hc = crc_w4(hc, hw2); hc = crc_w4(hc, hw3);
        hc = crc_w4(hc, (uint32_t)K); hc = crc_w4(hc, (uint32_t)(K >> 32));
        hc = crc_w4(hc, (uint32_t)poff); hc = crc_w4(hc, (uint32_t)(poff >> 32));
        hc = crc_w4(hc, (uint32_t)payload); hc = crc_w4(hc, (uint32_t)(payload >> 32));
        hc = crc_w4(hc, (uint32_t)ids_off); hc = crc_w4(hc, (uint32_t)(ids_off >> 32));
        hc = crc_w4(hc, (uint32_t)iend); hc = crc_w4(hc, (uint32_t)(iend >> 32));
        s_hc = hc;
    }
    __syncthreads();
    SMALL_STAMP(6);
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t w = 0; w < kSmallThreads / 32; ++w) acc ^= s_x[w];
        const uint32_t meta_crc = nwords == 0 ? 0u : (acc ^ 0xffffffffu);
        DevStats *st = a.st;
        st->K = K;
        st->total_units = K << (a.log2p - kSegLog2);
        st->poff = poff;
        st->payload_bytes = payload;
        st->ids_off = ids_off;
        st->image_bytes = ids_off + 4 * idsw;
        st->capacity = a.capacity;
        st->status = st->image_bytes > a.capacity ? kStCapacity : kStOk;
        st->img_flags = 0;
        st->n_regions = a.R;
        st->dirty_bytes = tot_bytes;
        st->dirty_runs = tot_runs;
        st->crc_acc = 0;
        st->meta_crc = meta_crc;
        const uint32_t hcrc = crc_w4(s_hc, meta_crc) ^ 0xffffffffu;
        uint4 *hd = reinterpret_cast<uint4 *>(img);
        hd[0] = make_uint4(hw0, hw1, hw2, hw3);
        hd[1] = make_uint4((uint32_t)K, (uint32_t)(K >> 32), (uint32_t)poff, (uint32_t)(poff >> 32));
        hd[2] = make_uint4((uint32_t)payload, (uint32_t)(payload >> 32), (uint32_t)ids_off, (uint32_t)(ids_off >> 32));
        hd[3] = make_uint4((uint32_t)iend, (uint32_t)(iend >> 32), meta_crc, hcrc);
    }
    small_leave(a, nw);
}

int small_blocks_per_sm() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_small_ckpt, kSmallThreads, 0) != cudaSuccess) {
        cudaGetLastError();
        n = 1;
    }
    return n > 0 ? n : 1;
}

void launch_small_ckpt(const Launch &L, const SmallArgs &a, int blocks) {
    // every CTA must be resident at once (grid barrier): a cooperative launch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.stream = L.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_small_ckpt, a);
    ++*L.counter;
}

int fused_blocks_per_sm() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_fused_compare, kFusedThreads, 0) != cudaSuccess) {
        cudaGetLastError();
        n = 2;
    }
    return n > 0 ? n : 1;
}

void launch_fused_compare(const Launch &L, const FusedArgs &a, int blocks) {
    // no more warps than tiles (every claim is an atomic on one counter)
    const uint64_t need = (a.n_tiles + kFusedThreads / 32 - 1) / (kFusedThreads / 32);
    if ((uint64_t)blocks > need) blocks = (int)(need ? need : 1);
    k_fused_compare<<<blocks, kFusedThreads, 0, L.stream>>>(a);
    ++*L.counter;
}


}  // namespace crum
