// kernels_zip.cu -- compressed images (DESIGN.md
// readings Z2-Z3).  The paper compresses the checkpoint image with gzip -1 or
// LZ4 on the CPU before writing it; here every 4 KiB
// payload unit is compressed on the GPU before it crosses the host link:
//   zero unit -> 0 bytes; else one DEFLATE block (RFC 1951, BFINAL = 1,
//   fixed Huffman codes) holding a greedy LZ77 parse, if shorter than the
//   unit; else the raw 4096 bytes.
// The parse (reading Z3): h(p) = (LE u32 at p * 2654435761) >> 20 for
// p <= 4092; cand(p) = the last q < p with h(q) == h(p), every position
// entering the table; len(p) = the longest run u[cand + i] == u[p + i],
// capped at min(258, 4096 - p); a match iff len >= 4; the parse is greedy
// from p = 0.
//
// One warp per unit:
//  1. hash candidates: 128 rounds of 32 consecutive positions; inside a round
//     __match_any_sync resolves equal hashes (the nearest lower lane wins),
//     across rounds a per-warp head table in shared memory.  A candidate whose
//     4 bytes match is "verified": exactly the positions where len >= 4, i.e.
//     where the greedy parse, if it stops there, emits a match.  Ballots give
//     a verified-candidate bitmap and a ">= 144" byte bitmap (9-bit literals).
//  2. greedy parse, warp-uniform: jump to the next verified candidate at or
//     after x (bitmap search), measure its match with all 32 lanes (8 bytes
//     each, first difference by a min-reduction), record it, x += len.  Match
//     lengths are computed only where the parse stops.
//  3. size: covered bitmap of the matches; literal bits = 8 per uncovered
//     position + 1 per uncovered byte >= 144; + the matches' bits.
//  4. emit, run by run: a literal run's bytes in parallel (bit offset of byte
//     i = 8 i + the >= 144 count before it, from prefix counts), then the
//     match; tokens are OR-ed into a shared-memory bit buffer (<= 2 words).
// Decoding is one warp per unit: lane 0 reads the symbols, writing literals
// and recording matches; the warp then expands the matches in order, each by
// all lanes (byte j of a match of distance d copies byte pos - d + j mod d,
// which precedes the match).
#include "crum_internal.cuh"

namespace crum {
namespace {

constexpr uint32_t kZHashShift = 20;        // 12-bit hash
constexpr uint32_t kZMaxMatch = 258;
constexpr uint32_t kZMinMatch = 4;
constexpr uint32_t kZEncWarps = 2;          // warps per encoder CTA
constexpr uint32_t kZEncCtasPerSm = 5;      // 10 warps / SM (22.5 KB of shared memory each)
constexpr uint32_t kZSeg = kSegBytes / 32;  // positions per lane segment
constexpr uint16_t kNone = 0xFFFF;

// Per-warp shared memory of the encoder.
constexpr uint32_t kZWords = kSegBytes / 32;  // 32-position bitmap words per unit

struct alignas(16) ZEncSmem {
    uint32_t data[kSegBytes / 4 + 4];  // the unit (+ 16 zero bytes for reads past the end)
    uint16_t head[kSegBytes];          // hash heads; then the output bits (as u32 words)
    uint16_t d[kSegBytes];             // distance of each position's verified candidate (0: none);
                                       // then the parse's matches, x | (len - 4) << 12 | (dist - 1) << 20,
                                       // as u32 words: match k overwrites d[2k], d[2k+1], entries of
                                       // positions the parse has passed (match k starts at >= 4k)
    uint32_t mcand[kZWords];           // bit p: position p has a verified candidate (a match >= 4)
    uint32_t m144[kZWords];            // bit p: byte p >= 144 (its literal code is 9 bits)
    uint32_t cov[kZWords];             // bit p: position p lies inside a match of the parse
    uint32_t p144[kZWords + 1];        // prefix counts of m144 words
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// 4 bytes at byte offset p of a word array (little-endian, unaligned).
__device__ __forceinline__ uint32_t ld32u(const uint32_t *w, uint32_t p) {
    const uint32_t lo = w[p >> 2], hi = w[(p >> 2) + 1];
    return __funnelshift_r(lo, hi, 8 * (p & 3));
}
__device__ __forceinline__ uint32_t byte_at(const uint32_t *w, uint32_t p) { return (w[p >> 2] >> (8 * (p & 3))) & 0xffu; }

// Huffman codes are written most significant bit first into an LSB-first stream.
__device__ __forceinline__ uint32_t rev(uint32_t code, uint32_t n) { return __brev(code) >> (32 - n); }

// Fixed literal/length code of symbol s (RFC 1951 sec. 3.2.6), bit-reversed; *n = bits.
__device__ __forceinline__ uint32_t litlen_bits(uint32_t s, uint32_t *n) {
    if (s <= 143) { *n = 8; return rev(0x30 + s, 8); }
    if (s <= 255) { *n = 9; return rev(0x190 + s - 144, 9); }
    if (s <= 279) { *n = 7; return rev(s - 256, 7); }
    *n = 8;
    return rev(0xC0 + s - 280, 8);
}

// A match (len 4..258, dist 1..4096) as one bit string (<= 31 bits): length
// code, its extra bits, 5-bit distance code, its extra bits (RFC 1951 3.2.5).
__device__ __forceinline__ uint32_t match_bits(uint32_t len, uint32_t dist, uint32_t *n) {
    uint32_t lsym, le = 0, lx = 0;
    if (len == kZMaxMatch) {
        lsym = 285;
    } else {
        const uint32_t v = len - 3;
        if (v < 8) {
            lsym = 257 + v;
        } else {
            le = (31 - __clz(v)) - 2;
            lsym = 257 + 4 * (le + 1) + ((v >> le) - 4);
            lx = v & ((1u << le) - 1);
        }
    }
    uint32_t dsym, de = 0, dx = 0;
    {
        const uint32_t v = dist - 1;
        if (v < 4) {
            dsym = v;
        } else {
            de = (31 - __clz(v)) - 1;
            dsym = 2 * (de + 1) + ((v >> de) - 2);
            dx = v & ((1u << de) - 1);
        }
    }
    uint32_t nl;
    uint32_t bits = litlen_bits(lsym, &nl);
    uint32_t k = nl;
    bits |= lx << k;
    k += le;
    bits |= rev(dsym, 5) << k;
    k += 5;
    bits |= dx << k;
    k += de;
    *n = k;
    return bits;
}

__device__ __forceinline__ uint32_t match_nbits(uint32_t len, uint32_t dist) {
    uint32_t n;
    match_bits(len, dist, &n);
    return n;
}

// OR n (<= 32) bits of v into the word buffer at bit position pos.
__device__ __forceinline__ void put_bits(uint32_t *out, uint32_t pos, uint32_t v, uint32_t n) {
    if (!n) return;
    const uint32_t w = pos >> 5, sh = pos & 31;
    atomicOr(out + w, v << sh);
    if (sh + n > 32) atomicOr(out + w + 1, v >> (32 - sh));
}

// >= 144 bytes at positions [0, x) (x <= 4096).
__device__ __forceinline__ uint32_t pre144(const ZEncSmem &sm, uint32_t x) {
    const uint32_t w = x >> 5, b = x & 31;
    return sm.p144[w] + (b ? __popc(sm.m144[w] & ((1u << b) - 1)) : 0u);
}

// Length of the match at y (distance dist, the first 4 bytes known equal),
// capped at cap: the first differing byte, found by all lanes (8 bytes each).
__device__ __forceinline__ uint32_t warp_match_len(const uint32_t *data, uint32_t y, uint32_t dist, uint32_t cap,
                                                   uint32_t lane) {
    for (uint32_t base = 0; base < cap; base += 256) {
        const uint32_t off = base + 8 * lane;
        uint32_t first = cap;  // this lane's first difference (or cap)
        if (off < cap) {
            const uint32_t a0 = ld32u(data, y + off), b0 = ld32u(data, y - dist + off);
            const uint32_t a1 = ld32u(data, y + off + 4), b1 = ld32u(data, y - dist + off + 4);
            uint32_t i = 8;
            if (a0 != b0) i = (__ffs(a0 ^ b0) - 1) >> 3;
            else if (a1 != b1) i = 4 + ((__ffs(a1 ^ b1) - 1) >> 3);
            first = min(cap, off + i);
            if (i == 8 && off + 8 < cap) first = cap;  // no difference here: a later lane decides
        }
        const uint32_t m = __reduce_min_sync(0xffffffffu, first);
        if (m < cap || base + 256 >= cap) return m;
    }
    return cap;
}

// ---------------------------------------------------------------------------
// Encoder: one warp per unit.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32 * kZEncWarps, kZEncCtasPerSm) k_zenc(const uint8_t *raw, uint64_t n,
                                                                          uint8_t *enc, uint16_t *zsz,
                                                                          const DevStats *st) {
    extern __shared__ __align__(16) uint8_t zsm_raw[];
    if (st->status == kStCorrupt) return;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    ZEncSmem &sm = reinterpret_cast<ZEncSmem *>(zsm_raw)[wid];
    const uint64_t nwarps = (uint64_t)gridDim.x * kZEncWarps;
    for (uint64_t u = (uint64_t)blockIdx.x * kZEncWarps + wid; u < n; u += nwarps) {
        {
            __syncwarp();  // the previous unit's readers of the shared buffers are done
            const uint4 *src = reinterpret_cast<const uint4 *>(raw + (u << kSegLog2));
            uint8_t *out_g = enc + (u << kSegLog2);
            // ---- load the unit ----
            uint32_t any = 0;
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) {
                const uint4 v = __ldcs(src + 32 * i + lane);  // read once: streaming
                reinterpret_cast<uint4 *>(sm.data)[32 * i + lane] = v;
                any |= v.x | v.y | v.z | v.w;
            }
            if (lane < 4) sm.data[kSegBytes / 4 + lane] = 0;
            if (!__any_sync(0xffffffffu, any != 0)) {
                if (lane == 0) zsz[u] = 0;  // zero unit: nothing to store
                continue;
            }
            // ---- 1. hash candidates, verified-candidate and >= 144 bitmaps ----
            for (uint32_t i = lane; i < kSegBytes / 2; i += 32) reinterpret_cast<uint32_t *>(sm.head)[i] = 0xFFFFFFFFu;
            __syncwarp();
            uint32_t found = 0;
            // rounds of 32 positions, four at a time: the hash work of the four
            // rounds is independent (its latency overlaps); only the table
            // reads / writes run round by round.  A round first assumes its 32
            // hashes are distinct: every lane takes the head entry as its
            // candidate and stores its position there, then reads the entry
            // back -- a lane that finds another lane's position shares its hash
            // with a lane of this round, and only then does the round resolve
            // its groups with __match_any_sync (the nearest lower lane of the
            // group is the candidate, the group's highest lane the new head).
            // MATCH.ANY costs hundreds of cycles; random data has a shared hash
            // in ~11 % of rounds (32 lanes, 4096 buckets).
            constexpr uint32_t kUnroll = 4;
            for (uint32_t c0 = 0; c0 < kZWords; c0 += kUnroll) {
                uint32_t v[kUnroll], h[kUnroll], q[kUnroll];
#pragma unroll
                for (uint32_t j = 0; j < kUnroll; ++j) {
                    const uint32_t p = 32 * (c0 + j) + lane;
                    v[j] = ld32u(sm.data, p);
                    h[j] = (v[j] * 2654435761u) >> kZHashShift;
                }
#pragma unroll
                for (uint32_t j = 0; j < kUnroll; ++j) {
                    const uint32_t p = 32 * (c0 + j) + lane;
                    const bool valid = p + 4 <= kSegBytes;
                    q[j] = valid ? sm.head[h[j]] : kNone;
                    __syncwarp();
                    if (valid) sm.head[h[j]] = (uint16_t)p;
                    __syncwarp();
                    const bool shared = valid && sm.head[h[j]] != (uint16_t)p;
                    if (__any_sync(0xffffffffu, shared)) {
                        const uint32_t peers = __match_any_sync(0xffffffffu, valid ? h[j] : 0x10000u + lane);
                        const uint32_t lower = peers & lanemask_lt();
                        if (valid && lower) q[j] = 32 * (c0 + j) + (31 - __clz(lower));
                        __syncwarp();
                        if (valid && (peers >> lane) == 1u) sm.head[h[j]] = (uint16_t)p;  // highest lane of its group
                    }
                    __syncwarp();
                }
#pragma unroll
                for (uint32_t j = 0; j < kUnroll; ++j) {
                    const uint32_t p = 32 * (c0 + j) + lane;
                    uint32_t dist = 0;
                    if (q[j] != kNone && ld32u(sm.data, q[j]) == v[j]) dist = p - q[j];  // 4 bytes match: len >= 4
                    sm.d[p] = (uint16_t)dist;
                    found |= dist;
                    const uint32_t mc = __ballot_sync(0xffffffffu, dist != 0);
                    const uint32_t mb = __ballot_sync(0xffffffffu, (v[j] & 0xffu) >= 144);
                    if (lane == 0) {
                        sm.mcand[c0 + j] = mc;
                        sm.m144[c0 + j] = mb;
                    }
                }
                __syncwarp();
            }
            if (!__any_sync(0xffffffffu, found != 0)) {
                // no match anywhere: >= 8 bits per byte, the unit stays raw
#pragma unroll
                for (uint32_t i = 0; i < 8; ++i)
                    reinterpret_cast<uint4 *>(out_g)[32 * i + lane] = reinterpret_cast<const uint4 *>(sm.data)[32 * i + lane];
                if (lane == 0) zsz[u] = (uint16_t)kSegBytes;
                continue;
            }
            // ---- 2. greedy parse (warp-uniform) ----
            uint32_t *match = reinterpret_cast<uint32_t *>(sm.d);
            uint32_t nm = 0;
            for (uint32_t x = 0; x < kSegBytes;) {
                uint32_t w = x >> 5;
                uint32_t m = sm.mcand[w] & (0xFFFFFFFFu << (x & 31));
                if (!m) {
                    bool hit = false;
                    for (uint32_t b = w + 1; b < kZWords; b += 32) {
                        const uint32_t wi = b + lane;
                        const uint32_t mm = wi < kZWords ? sm.mcand[wi] : 0u;
                        const uint32_t bal = __ballot_sync(0xffffffffu, mm != 0);
                        if (bal) {
                            const uint32_t f = __ffs(bal) - 1;
                            w = b + f;
                            m = __shfl_sync(0xffffffffu, mm, f);
                            hit = true;
                            break;
                        }
                    }
                    if (!hit) break;
                }
                const uint32_t y = 32 * w + (__ffs(m) - 1);
                const uint32_t dist = sm.d[y];
                const uint32_t L = warp_match_len(sm.data, y, dist, min(kZMaxMatch, kSegBytes - y), lane);
                if (lane == 0) match[nm] = y | ((L - kZMinMatch) << 12) | ((dist - 1) << 20);
                ++nm;
                x = y + L;
            }
            __syncwarp();
            // ---- 3. size: covered positions, literal and match bits ----
            for (uint32_t i = lane; i < kZWords; i += 32) sm.cov[i] = 0;
            __syncwarp();
            uint32_t mbits = 0;
            for (uint32_t i = lane; i < nm; i += 32) {
                const uint32_t mr = match[i];
                const uint32_t x0 = mr & 0xfffu, x1 = x0 + ((mr >> 12) & 0xffu) + kZMinMatch;
                mbits += match_nbits(x1 - x0, (mr >> 20) + 1);
                for (uint32_t wq = x0 >> 5; wq <= (x1 - 1) >> 5; ++wq) {
                    const uint32_t lo = max(x0, 32 * wq) - 32 * wq, hi = min(x1, 32 * wq + 32) - 32 * wq;
                    const uint32_t bits = (hi == 32 ? 0xFFFFFFFFu : ((1u << hi) - 1)) & ~((1u << lo) - 1);
                    atomicOr(&sm.cov[wq], bits);
                }
            }
            __syncwarp();
            uint32_t nlit = 0, n144 = 0, c144[kZWords / 32];
#pragma unroll
            for (uint32_t k = 0; k < kZWords / 32; ++k) {
                const uint32_t wq = 4 * lane + k;  // lane owns 4 consecutive words (prefix counts below)
                const uint32_t lit = ~sm.cov[wq];
                nlit += __popc(lit);
                n144 += __popc(lit & sm.m144[wq]);
                c144[k] = __popc(sm.m144[wq]);
            }
            const uint32_t total = 3 + 8 * __reduce_add_sync(0xffffffffu, nlit) + __reduce_add_sync(0xffffffffu, n144) +
                                   __reduce_add_sync(0xffffffffu, mbits) + 7;
            const uint32_t nbytes = (total + 7) / 8;
            if (nbytes >= kSegBytes) {
#pragma unroll
                for (uint32_t i = 0; i < 8; ++i)
                    reinterpret_cast<uint4 *>(out_g)[32 * i + lane] = reinterpret_cast<const uint4 *>(sm.data)[32 * i + lane];
                if (lane == 0) zsz[u] = (uint16_t)kSegBytes;
                continue;
            }
            {   // prefix counts of the >= 144 bitmap (4 words per lane, warp scan)
                const uint32_t own = c144[0] + c144[1] + c144[2] + c144[3];
                uint32_t inc = own;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= (uint32_t)o) inc += y;
                }
                uint32_t run = inc - own;
#pragma unroll
                for (uint32_t k = 0; k < kZWords / 32; ++k) {
                    sm.p144[4 * lane + k] = run;
                    run += c144[k];
                }
                if (lane == 31) sm.p144[kZWords] = run;
            }
            // ---- 4. emit, run by run ----
            uint32_t *obits = reinterpret_cast<uint32_t *>(sm.head);  // the hash heads are no longer needed
            const uint32_t nwords = (nbytes + 15) / 16 * 4;         // whole 16-byte rows
            for (uint32_t i = lane; i < nwords + 1; i += 32) obits[i] = 0;
            __syncwarp();
            if (lane == 0) put_bits(obits, 0, 3u, 3);  // BFINAL = 1, BTYPE = 01
            uint32_t pos = 3, s0 = 0;
            for (uint32_t mi = 0; mi <= nm; ++mi) {
                uint32_t x1 = kSegBytes, L = 0, dist = 0;
                if (mi < nm) {
                    const uint32_t mr = match[mi];
                    x1 = mr & 0xfffu;
                    L = ((mr >> 12) & 0xffu) + kZMinMatch;
                    dist = (mr >> 20) + 1;
                }
                const uint32_t b144 = pre144(sm, s0);
                for (uint32_t i = lane; i < x1 - s0; i += 32) {
                    const uint32_t xp = s0 + i;
                    uint32_t n;
                    const uint32_t v = litlen_bits(byte_at(sm.data, xp), &n);
                    put_bits(obits, pos + 8 * i + (pre144(sm, xp) - b144), v, n);
                }
                pos += 8 * (x1 - s0) + (pre144(sm, x1) - b144);
                if (mi < nm) {
                    uint32_t n;
                    const uint32_t v = match_bits(L, dist, &n);
                    if (lane == 0) put_bits(obits, pos, v, n);
                    pos += n;
                    s0 = x1 + L;
                }
            }
            // end of block: code 256 is seven zero bits
            __syncwarp();
            for (uint32_t i = lane; i < nwords / 4; i += 32)
                reinterpret_cast<uint4 *>(out_g)[i] = reinterpret_cast<const uint4 *>(obits)[i];
            if (lane == 0) zsz[u] = (uint16_t)nbytes;
        }
    }
}

// ---------------------------------------------------------------------------
// Chunk scan: one block of 1024 threads, <= kZChunkUnits units.
// ---------------------------------------------------------------------------
constexpr uint32_t kZScanPer = kZChunkUnits / 1024;  // units per thread

// Exclusive offsets of the n (<= kZChunkUnits) sizes of one chunk (zloc,
// chunk-relative); *zbase = the running total before the chunk, *zrun and
// *zrun_host (mapped, nullable) = after it.
__global__ void __launch_bounds__(1024) k_zscan_chunk(const uint16_t *zsz, uint64_t n, uint32_t *zloc,
                                                      uint64_t *zrun, uint64_t *zbase, uint64_t *zrun_host) {
    const uint64_t run = *zrun;
    uint32_t v[kZScanPer];
    uint64_t sum = 0;
#pragma unroll
    for (uint32_t j = 0; j < kZScanPer; ++j) {
        const uint64_t i = threadIdx.x * kZScanPer + j;
        v[j] = i < n ? zsz[i] : 0u;
        sum += v[j];
    }
    uint64_t tot;
    uint64_t o = block_excl_scan(sum, &tot);
#pragma unroll
    for (uint32_t j = 0; j < kZScanPer; ++j) {
        const uint64_t i = threadIdx.x * kZScanPer + j;
        if (i < n) zloc[i] = (uint32_t)o;
        o += v[j];
    }
    if (threadIdx.x == 0) {
        *zbase = run;
        *zrun = run + tot;
        if (zrun_host) *reinterpret_cast<volatile uint64_t *>(zrun_host) = run + tot;
    }
}

// ---------------------------------------------------------------------------
// Pack: one warp per unit, byte-exact destination:
// dst + (base ? *base : 0) + zloc[i]; limit != 0: a unit is written only if
// that payload offset + its size <= limit (the payload bytes that fit).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_zpack(const uint8_t *stage, const uint16_t *zsz, const uint32_t *zloc,
                                               uint64_t n, const uint64_t *base, uint8_t *dst, uint64_t limit,
                                               const DevStats *st) {
    if (st->status == kStCorrupt) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t b = base ? *base : 0;
    for (uint64_t u = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        const uint32_t sz = zsz[u];
        if (!sz) continue;
        const uint64_t off = b + zloc[u];
        if (limit && off + sz > limit) continue;  // does not fit: CAPACITY at the end
        const uint32_t *s = reinterpret_cast<const uint32_t *>(stage + (u << kSegLog2));
        uint8_t *d = dst + off;
        // head bytes up to a 4-byte boundary of the destination, whole words, tail bytes
        const uint32_t head = (uint32_t)((4 - (reinterpret_cast<uintptr_t>(d) & 3)) & 3);
        const uint32_t h = min(head, sz);
        if (lane < h) d[lane] = (uint8_t)(s[lane >> 2] >> (8 * (lane & 3)));
        const uint32_t nw = (sz - h) / 4;
        uint32_t *dw = reinterpret_cast<uint32_t *>(d + h);
        // destination word i holds source bytes h + 4 i ..: words h / 4 + i
        // (h <= 3, so word i) and i + 1 shifted by 8 h; the next word only when
        // h != 0 (then it holds bytes of this encoding; otherwise it may lie
        // past what was written).  Eight loads in flight per lane before the
        // stores: a 4 KiB unit is 4 round trips to L2, not 32.
        const uint32_t sh = 8 * (h & 3);
        for (uint32_t i0 = 0; i0 < nw; i0 += 32 * 8) {
            uint32_t lo[8], hi[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                lo[k] = i < nw ? s[i] : 0u;
                hi[k] = (i < nw && sh) ? s[i + 1] : 0u;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t i = i0 + 32 * k + lane;
                if (i < nw) dw[i] = __funnelshift_r(lo[k], hi[k], sh);
            }
        }
        const uint32_t t0 = h + 4 * nw;
        if (t0 + lane < sz) {
            const uint32_t p = t0 + lane;
            d[p] = (uint8_t)(s[p >> 2] >> (8 * (p & 3)));
        }
    }
}

// After the last chunk: the compressed image's fields (as the gather branch
// of the plain path's finalisation) and the payload's zero padding.
__global__ void __launch_bounds__(256) k_zfinal(DevStats *st, const uint64_t *zrun, uint8_t *img, uint64_t capacity) {
    if (st->status != kStOk) return;
    const uint64_t Z = *zrun, zpay = round_up(Z, kSegBytes);
    const uint64_t K = st->K, U = st->total_units;
    const uint64_t ids_off = st->poff + zpay;
    const uint64_t image = ids_off + round_up(4 * K, 8) + ((st->img_flags & 2u) ? 8 * K : 0) + round_up(2 * U, 8);
    __syncthreads();
    if (threadIdx.x == 0) {
        st->payload_bytes = zpay;
        st->ids_off = ids_off;
        st->image_bytes = image;
        st->img_flags |= 4u;
        if (image > capacity) st->status = kStCapacity;
    }
    if (img && image <= capacity)
        for (uint64_t b = st->poff + Z + threadIdx.x; b < st->poff + zpay; b += blockDim.x) img[b] = 0;
}

// ---------------------------------------------------------------------------
// Restore: size table validation + offsets (all units).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_zscan_local(const uint16_t *zsz, DevStats *st, uint32_t *zloc,
                                                    uint64_t *zblk) {
    const uint64_t U = st->total_units;
    const uint64_t base = (uint64_t)blockIdx.x * kZScanBlock;
    if (base >= U) return;
    constexpr uint32_t per = kZScanBlock / 256;
    uint32_t v[per];
    uint64_t sum = 0;
    bool bad = false;
#pragma unroll
    for (uint32_t j = 0; j < per; ++j) {
        const uint64_t u = base + threadIdx.x * per + j;
        v[j] = u < U ? zsz[u] : 0u;
        bad |= v[j] > kSegBytes;
        sum += v[j];
    }
    uint64_t tot;
    uint64_t ex = block_excl_scan(sum, &tot);
#pragma unroll
    for (uint32_t j = 0; j < per; ++j) {
        const uint64_t u = base + threadIdx.x * per + j;
        if (u < U) zloc[u] = (uint32_t)ex;
        ex += v[j];
    }
    if (threadIdx.x == 0) zblk[blockIdx.x] = tot;
    if (bad) st->status = kStCorrupt;
}

// Exclusive scan of the block totals (one block); the sizes must sum to the
// header's payload length before its zero padding, and the size table's
// padding must be zero.
__global__ void __launch_bounds__(1024) k_zscan_top(uint64_t *zblk, DevStats *st, const uint16_t *zsz) {
    const uint64_t U = st->total_units;
    const uint64_t nblk = (U + kZScanBlock - 1) / kZScanBlock;
    uint64_t carry = 0;
    for (uint64_t b0 = 0; b0 < nblk; b0 += blockDim.x) {
        const uint64_t b = b0 + threadIdx.x;
        const uint64_t v = b < nblk ? zblk[b] : 0;
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, &tot);
        if (b < nblk) zblk[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) {
        zblk[nblk] = carry;
        bool bad = round_up(carry, kSegBytes) != st->payload_bytes;
        for (uint64_t q = U; q < round_up(U, 4); ++q) bad |= zsz[q] != 0;
        if (bad) st->status = kStCorrupt;
    }
}

// ---------------------------------------------------------------------------
// Decoder: one warp per unit.
// ---------------------------------------------------------------------------
constexpr uint32_t kZDecWarps = 8;
// Any valid stream: matches are >= 3 bytes (RFC 1951), so <= 1365 of them fill a unit.
constexpr uint32_t kZMaxMatches = kSegBytes / 3 + 1;

struct alignas(16) ZDecSmem {
    uint32_t in[kSegBytes / 4 + 4];  // the encoded bytes (shifted by the source's misalignment)
    uint32_t out[kSegBytes / 4];
    uint32_t match[kZMaxMatches];    // pos | (len - 3) << 12 | (dist - 1) << 20
};

// RFC 1951 sec. 3.2.5 bases (lengths 257..285 and distances 0..29).
__constant__ uint16_t c_len_base[29] = {3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31,
                                        35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2,
                                        3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dist_base[30] = {1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193,
                                         257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145,
                                         8193, 12289, 16385, 24577};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6,
                                         7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

// LSB-first bit reader over shared memory words, starting at bit `pos`.
struct BitIn {
    const uint32_t *w;
    uint32_t pos, end;  // bit positions
    __device__ __forceinline__ uint32_t peek(uint32_t n) const {  // n <= 25
        const uint32_t q = pos >> 5, sh = pos & 31;
        const uint64_t x = ((uint64_t)w[q + 1] << 32) | w[q];
        return (uint32_t)(x >> sh) & ((1u << n) - 1);
    }
    __device__ __forceinline__ uint32_t get(uint32_t n) {
        const uint32_t v = n ? peek(n) : 0u;
        pos += n;
        return v;
    }
};

__global__ void __launch_bounds__(32 * kZDecWarps, 2) k_zinflate(const uint8_t *src, const uint16_t *zsz,
                                                                  const uint32_t *zloc, const uint64_t *zblk,
                                                                  DevStats *st, uint8_t *dst, uint64_t u_lo,
                                                                  uint64_t u_hi, int rebase) {
    extern __shared__ __align__(16) uint8_t zdsm_raw[];
    if (st->status != kStOk) return;
    const uint64_t U = min(u_hi, st->total_units);
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    ZDecSmem &sm = reinterpret_cast<ZDecSmem *>(zdsm_raw)[wid];
    const uint64_t off0 = rebase ? ((zblk[u_lo / kZScanBlock] + zloc[u_lo]) & ~3ull) : 0;
    const uint64_t nwarps = (uint64_t)gridDim.x * kZDecWarps;
    for (uint64_t u = u_lo + (uint64_t)blockIdx.x * kZDecWarps + wid; u < U; u += nwarps) {
        const uint32_t n = zsz[u];
        const uint64_t off = zblk[u / kZScanBlock] + zloc[u] - off0;
        uint4 *out_g = dst ? reinterpret_cast<uint4 *>(dst + ((u - u_lo) << kSegLog2)) : nullptr;
        if (n == 0) {
            if (out_g)
                for (uint32_t i = lane; i < kSegBytes / 16; i += 32) out_g[i] = make_uint4(0, 0, 0, 0);
            continue;
        }
        if (n > kSegBytes) {  // validated by the size scan already
            if (lane == 0) st->status = kStCorrupt;
            continue;
        }
        // stage the encoded bytes: aligned words covering [off, off + n)
        const uint32_t mis = (uint32_t)(off & 3);
        const uint32_t *sw = reinterpret_cast<const uint32_t *>(src + (off - mis));
        const uint32_t nw = (mis + n + 3) / 4;
        for (uint32_t i = lane; i < nw; i += 32) sm.in[i] = sw[i];
        if (lane < 2) sm.in[nw + lane] = 0;
        __syncwarp();
        if (n == kSegBytes) {  // raw unit
            if (out_g)
                for (uint32_t i = lane; i < kSegBytes / 4; i += 32)
                    reinterpret_cast<uint32_t *>(out_g)[i] = __funnelshift_r(sm.in[i], sm.in[i + 1], 8 * mis);
            __syncwarp();
            continue;
        }
        // ---- lane 0: the symbols ----
        uint32_t ok = 1, nm = 0;
        if (lane == 0) {
            uint8_t *ob = reinterpret_cast<uint8_t *>(sm.out);
            BitIn b{sm.in, 8 * mis, 8 * mis + 8 * n};
            ok = b.get(1) == 1 && b.get(2) == 1;  // BFINAL = 1, BTYPE = 01
            uint32_t o = 0;
            while (ok) {
                if (b.pos + 7 > b.end) { ok = 0; break; }
                // the next 9 bits, most significant code bit first
                const uint32_t c9 = __brev(b.peek(9)) >> 23;
                uint32_t sym;
                if ((c9 >> 2) <= 0x17) {
                    sym = 256 + (c9 >> 2);
                    b.pos += 7;
                } else if ((c9 >> 1) <= 0xBF) {
                    sym = (c9 >> 1) - 0x30;
                    b.pos += 8;
                } else if ((c9 >> 1) <= 0xC7) {
                    sym = 280 + (c9 >> 1) - 0xC0;
                    b.pos += 8;
                } else {
                    sym = 144 + c9 - 0x190;
                    b.pos += 9;
                }
                if (b.pos > b.end || sym >= 286) { ok = 0; break; }
                if (sym == 256) break;
                if (sym < 256) {
                    if (o >= kSegBytes) { ok = 0; break; }
                    ob[o++] = (uint8_t)sym;
                    continue;
                }
                const uint32_t lc = sym - 257;
                const uint32_t len = c_len_base[lc] + b.get(c_len_extra[lc]);
                const uint32_t dc = __brev(b.get(5)) >> 27;
                if (dc >= 30 || b.pos > b.end) { ok = 0; break; }
                const uint32_t dist = c_dist_base[dc] + b.get(c_dist_extra[dc]);
                if (b.pos > b.end || dist > o || o + len > kSegBytes || nm >= kZMaxMatches) { ok = 0; break; }
                sm.match[nm++] = o | ((len - 3) << 12) | ((dist - 1) << 20);
                o += len;
            }
            // exactly 4096 bytes; the stream ends in its last byte, zero padding bits
            if (ok && o != kSegBytes) ok = 0;
            if (ok && (b.pos + 7) / 8 != 8 * mis / 8 + n) ok = 0;
            if (ok && b.pos < b.end && b.peek(b.end - b.pos) != 0) ok = 0;
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        nm = __shfl_sync(0xffffffffu, nm, 0);
        if (!ok) {
            if (lane == 0) st->status = kStCorrupt;
            continue;
        }
        __syncwarp();
        if (!out_g) continue;  // validation only
        // ---- the warp: matches in order (each reads only bytes before it) ----
        uint8_t *ob = reinterpret_cast<uint8_t *>(sm.out);
        for (uint32_t m = 0; m < nm; ++m) {
            const uint32_t mr = sm.match[m];
            const uint32_t pos = mr & 0xfffu, len = ((mr >> 12) & 0xffu) + 3, dist = (mr >> 20) + 1;
            if (dist >= len) {
                for (uint32_t j = lane; j < len; j += 32) ob[pos + j] = ob[pos - dist + j];
            } else {
                for (uint32_t j = lane; j < len; j += 32) ob[pos + j] = ob[pos - dist + j % dist];
            }
            __syncwarp();
        }
        for (uint32_t i = lane; i < kSegBytes / 16; i += 32) out_g[i] = reinterpret_cast<const uint4 *>(sm.out)[i];
        __syncwarp();
    }
}

// Copy payload bytes [off(u_lo) & ~3, round_up(end(u_hi - 1), 4)) from src
// (e.g. a pinned image's mapped address) into dst, wide and coalesced.
__global__ void __launch_bounds__(256) k_zfetch(const uint8_t *src, const uint16_t *zsz, const uint32_t *zloc,
                                               const uint64_t *zblk, uint64_t u_lo, uint64_t u_hi, uint8_t *dst) {
    if (u_hi <= u_lo) return;
    const uint64_t b0 = (zblk[u_lo / kZScanBlock] + zloc[u_lo]) & ~3ull;
    const uint64_t b1 = round_up(zblk[(u_hi - 1) / kZScanBlock] + zloc[u_hi - 1] + zsz[u_hi - 1], 4);
    const uint64_t n4 = (b1 - b0) / 4;
    const uint32_t *s4 = reinterpret_cast<const uint32_t *>(src + b0);
    uint32_t *d4 = reinterpret_cast<uint32_t *>(dst);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        const uint32_t a = s4[i], b = s4[i + stride], c = s4[i + 2 * stride], d = s4[i + 3 * stride];
        d4[i] = a;
        d4[i + stride] = b;
        d4[i + 2 * stride] = c;
        d4[i + 3 * stride] = d;
    }
    for (; i < n4; i += stride) d4[i] = s4[i];
}

unsigned z_grid(const Launch &L, uint64_t units, uint32_t warps_per_block, uint32_t blocks_per_sm) {
    uint64_t blocks = (units + warps_per_block - 1) / warps_per_block;
    const uint64_t cap = (uint64_t)L.sms * blocks_per_sm;
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks ? blocks : 1);
}

}  // namespace

void launch_zenc(const Launch &L, const uint8_t *raw, uint64_t n, uint8_t *enc, uint16_t *zsz, const DevStats *st) {
    if (!n) return;
    const size_t smem = sizeof(ZEncSmem) * kZEncWarps;
    cudaFuncSetAttribute(k_zenc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_zenc<<<z_grid(L, n, kZEncWarps, kZEncCtasPerSm), 32 * kZEncWarps, smem, L.stream>>>(raw, n, enc, zsz, st);
    ++*L.counter;
}

void launch_zscan_chunk(const Launch &L, const uint16_t *zsz, uint64_t n, uint32_t *zloc, uint64_t *zrun,
                        uint64_t *zbase, uint64_t *zrun_host) {
    k_zscan_chunk<<<1, 1024, 0, L.stream>>>(zsz, n, zloc, zrun, zbase, zrun_host);
    ++*L.counter;
}

void launch_zpack(const Launch &L, const uint8_t *stage, const uint16_t *zsz, const uint32_t *zloc, uint64_t n,
                  const uint64_t *base, uint8_t *dst, uint64_t limit, const DevStats *st) {
    if (!n) return;
    k_zpack<<<z_grid(L, n, 8, 8), 256, 0, L.stream>>>(stage, zsz, zloc, n, base, dst, limit, st);
    ++*L.counter;
}

void launch_zfinal(const Launch &L, DevStats *st, const uint64_t *zrun, uint8_t *img, uint64_t capacity) {
    k_zfinal<<<1, 256, 0, L.stream>>>(st, zrun, img, capacity);
    ++*L.counter;
}

void launch_zscan(const Launch &L, const uint16_t *zsz, DevStats *st, uint32_t *zloc, uint64_t *zblk,
                  uint64_t max_units) {
    const uint64_t nblk = (max_units + kZScanBlock - 1) / kZScanBlock;
    k_zscan_local<<<(unsigned)(nblk ? nblk : 1), 256, 0, L.stream>>>(zsz, st, zloc, zblk);
    k_zscan_top<<<1, 1024, 0, L.stream>>>(zblk, st, zsz);
    *L.counter += 2;
}

void launch_zdecode(const Launch &L, const uint8_t *src, const uint16_t *zsz, const uint32_t *zloc,
                    const uint64_t *zblk, DevStats *st, uint8_t *dst, uint64_t units, uint64_t u_lo, int rebase) {
    if (!units) return;
    const size_t smem = sizeof(ZDecSmem) * kZDecWarps;
    cudaFuncSetAttribute(k_zinflate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_zinflate<<<z_grid(L, units, kZDecWarps, 2), 32 * kZDecWarps, smem, L.stream>>>(src, zsz, zloc, zblk, st, dst,
                                                                                    u_lo, u_lo + units, rebase);
    ++*L.counter;
}

void launch_zfetch(const Launch &L, const uint8_t *src, const uint16_t *zsz, const uint32_t *zloc,
                   const uint64_t *zblk, uint64_t u_lo, uint64_t u_hi, uint8_t *dst) {
    if (u_hi <= u_lo) return;
    uint64_t blocks = ((u_hi - u_lo) * 1024 + 255) / 256;
    if (blocks > (uint64_t)L.sms * 8) blocks = L.sms * 8;
    k_zfetch<<<(unsigned)(blocks ? blocks : 1), 256, 0, L.stream>>>(src, zsz, zloc, zblk, u_lo, u_hi, dst);
    ++*L.counter;
}

}  // namespace crum
