// crum_internal.cuh -- device-side data layout and kernel launchers of
// libcrum.so (private to the library; the ABI is include/crum.h).
//
// HBM layout:
//   * registered regions: the caller's bytes, untouched except by restore.
//   * per region: COMPARE -> byte mirror (B_r bytes, 256-B aligned);
//                 HASH    -> u64 table[n_r] (last committed XXH3 per page).
//   * per context, indexed by the global page id g (regions ascending, pages
//     ascending; page i of region r is g = page_base_r + i):
//       force[g]   u8  force-dirty bit (register sets all; commit clears)
//       flags[g]   u8  "content changed" bit written by detect (scratch)
//       newhash[g] u64 XXH3 of the page computed by detect (scratch)
//       gids[K]    u32 compacted dirty page ids, ascending (scratch)
//     per-page arrays are padded to a multiple of kPagesPerCompactBlock with
//     zeros so compaction can use 16-byte vector loads without bounds checks.
//   * image (device buffer): v1 format, header | table | ids | hashes | pad |
//     payload (slots of P_r bytes, 4096-aligned).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/crum.h"

namespace crum {

constexpr uint32_t kSegLog2 = 12;              // 4 KiB work segment (min page size)
constexpr uint32_t kSegBytes = 1u << kSegLog2;
constexpr uint32_t kU2sDirectLog2 = 4;         // compaction: pages of <= 16 units write their unit->slot entries inline
constexpr uint32_t kPagesPerThread = 16;       // compaction: one uint4 of flags per thread
constexpr uint32_t kCompactThreads = 256;
constexpr uint32_t kPagesPerCompactBlock = kPagesPerThread * kCompactThreads;  // 4096

enum : uint32_t { kModeCompare = 0, kModeHash = 1, kModeTracked = 2 };
enum : uint32_t { kStOk = 0, kStCapacity = 6, kStCorrupt = 7 };

struct DevRegion {
    uint8_t *base;      // registered bytes
    uint8_t *mirror;    // compare mode snapshot (nullptr in hash mode)
    uint64_t *table;    // hash mode snapshot (nullptr in compare mode)
    uint64_t bytes;     // B_r
    uint64_t page_base; // global id of page 0
    uint64_t n_pages;   // n_r
    uint32_t log2p;     // log2(P_r)
    uint32_t mode;
    uint32_t id;
    uint32_t aligned32; // base is 32-byte aligned (256-bit vector path allowed)
};

// Per-region results of compaction (gather) or of the image table (restore).
struct RegStat {
    uint64_t first;        // index of the region's first listed slot
    uint64_t n_dirty;      // slots listed for the region
    uint64_t payload_base; // byte offset of the region's first slot inside the payload
    uint64_t unit_base;    // 4 KiB payload units before the region (prefix)
};

// Device-resident bookkeeping of one gather / restore call.
struct DevStats {
    uint64_t K;
    uint64_t poff;           // payload offset = round_up(64 + 48R, 4096)
    uint64_t payload_bytes;
    uint64_t ids_off;        // poff + payload_bytes
    uint64_t image_bytes;
    uint64_t dirty_bytes;
    uint64_t dirty_runs;
    uint64_t total_units;    // payload_bytes / 4096
    uint64_t capacity;       // device image capacity (gather)
    uint32_t status;         // kStOk / kStCapacity / kStCorrupt
    uint32_t crc_acc;        // XOR of per-chunk raw CRC terms (meta CRC)
    uint32_t img_flags;      // header flags (bit0 FULL, bit1 HAS_HASHES, bit2 COMPRESSED)
    uint32_t n_regions;
    uint32_t meta_crc;       // final zlib CRC-32 of table || ids || hashes
    uint32_t pad0;
    uint64_t t_ns;           // small path, timed: first CTA in -> last CTA out (globaltimer ns)
};

// Running totals of the compaction before range c (rb[c]); rb[0] = {0, 0}.
struct RangeTotals {
    uint64_t k;
    uint64_t units;
};

struct X2N {
    uint32_t t[32];   // x^(2^k) mod P (reflected CRC-32 polynomial)
    uint32_t pw[32];  // x^(8 * 64 * j) mod P: shift by j 64-byte chunks
    uint32_t lpw[32]; // x^(8 * 16 * j) mod P: shift by j 16-byte chunks
    uint32_t wpw[8];  // x^(8 * 512 * w) mod P: shift by w warps of 16-byte chunks
};

struct Launch {
    cudaStream_t stream;
    int sms;
    uint64_t *counter;  // incremented per kernel launch
};

// A2: compaction of pages [p_lo, p_hi) (p_lo % 16 == 0), range index c.
struct CompactArgs {
    uint8_t *flags;        // detect marks (== tag); the write pass clears its range's bytes
    const uint8_t *force;
    const DevRegion *regs;
    const uint64_t *newhash;
    uint64_t p_lo, p_hi;
    uint32_t R;
    uint32_t tag;          // flags[g] == tag <=> content changed in this checkpoint
    int full;              // CRUM_FULL: every page listed
    int has_hashes;
    int first_range;       // reset per-checkpoint accumulators
    int final_range;       // finalise: region prefix sums, header fields, table
    uint32_t c;
    uint64_t *blk_units;   // per-block 4 KiB units
    uint32_t *gids;        // slot -> global page id
    uint64_t *sunit;       // slot -> payload unit offset
    uint32_t *u2s;         // payload unit -> slot (every unit of every listed page)
    uint32_t *lids;        // slot -> region-local page id (image ids)
    uint64_t *lhash;       // slot -> XXH3 (hash regions) or 0 (image hashes)
    uint32_t *reg_nd;      // per-region dirty count
    RangeTotals *rb;
    RangeTotals *rb_host;  // mapped pinned mirror of rb (host reads it after an event)
    uint32_t *done;        // last-block counter (self-resetting)
    RegStat *rs;
    DevStats *st;
    uint64_t capacity;
    uint8_t *head;         // image head (header + table + pad) or nullptr
};

// A3: gather units [u_lo, u_hi) of the range with totals rb[0] (before) and
// rb[1] (after).  dst == nullptr: commit only.  Unit u is written at
// dst + (add_poff ? st->poff : 0) + (u - dst_unit0) * 4096.
struct GatherArgs {
    const DevRegion *regs;
    uint32_t R;
    int add_poff;
    const uint32_t *gids;
    const uint64_t *sunit;
    const uint32_t *u2s;
    const uint64_t *newhash;
    const RangeTotals *rb;
    const DevStats *st;
    uint8_t *dst;
    uint64_t dst_unit0;
    uint8_t *force;
    uint64_t u_lo, u_hi;
    int no_commit;  // 1: copy to dst only (the commit runs later as a dst == nullptr pass)
};

// Metadata CRC + tail copy + header (last block).
struct CrcArgs {
    uint8_t *head;          // header + table (table already written)
    uint8_t *tail;          // ids/hashes destination, nullptr: head + st->ids_off
    const uint32_t *lids;
    const uint64_t *lhash;
    const uint32_t *gids;
    DevStats *st;
    DevStats *st_host;      // mapped pinned copy of the final stats, or nullptr
    uint32_t *done;
    X2N x2n;
    const uint16_t *zsz;    // compressed image: per-unit encoded sizes (tail after the hashes)
    uint8_t *out;           // nullptr, or the image's mapped address: the table + padding
                            // [64, poff) are copied there from head, the tail and header go there
};

// A6: scatter units [u_lo, u_hi); unit u read from src + (u - src_unit0)*4096.
struct ScatterArgs {
    const DevRegion *regs;
    uint32_t R;
    const RegStat *rs;
    const uint32_t *ids;
    const uint64_t *hashes;
    const DevStats *st;
    const uint8_t *src;
    uint64_t src_unit0;
    uint8_t *force;
    uint64_t u_lo, u_hi;
    const uint8_t *skip;   // lazy restore: slots with skip[k] != 0 are left alone (may be null)
    uint8_t *mark;         // lazy restore: mark[k] = 1 for every slot written (may be null;
                           // never the same array as skip within one launch)
};

// Single-pass checkpoint (all regions COMPARE, P <= 64 KiB): detect +
// decoupled look-back compaction + gather + commit in one persistent kernel.
constexpr uint32_t kFusedMaxLog2P = 16;
constexpr uint32_t kFusedMinTileLog2 = 15;   // tile = max(P, 32 KiB) (footprints above kFusedSmallBytes)
constexpr uint64_t kFusedSmallBytes = 64ull << 20;  // at or below: tile = one page, metadata CRC in-kernel
constexpr uint32_t kFusedInlineMeta = 16384;        // in-kernel CRC when table + ids can reach at most this
struct FusedScratch {
    uint32_t ticket;          // next tile to claim
    uint32_t done;            // tiles finished
    uint64_t dirty_bytes;     // accumulated logical bytes of listed pages
};
// One contiguous scratch per context, cleared by ONE memset before every
// launch: FusedScratch | per-region counts | look-back status words.
struct FusedArgs {
    const DevRegion *regs;
    uint32_t R;
    uint32_t tag;             // tag of the look-back status words (constant: they are cleared per launch)
    uint32_t tile_log2_min;   // tile = max(P, 2^tile_log2_min) bytes
    int inline_meta;          // the finalising warp writes tail, runs, CRC and header (no k_crc_meta)
    X2N x2n;                  // CRC shift tables (inline_meta)
    const uint64_t *tile_base;// per region: first tile (prefix, R + 1 entries)
    uint64_t n_tiles;
    uint64_t *status;         // per tile: tag | state | count | units
    FusedScratch *fs;
    uint8_t *force;
    uint8_t *img;             // device image (payload at poff)
    uint8_t *meta;            // nullptr, or where the region table + padding go instead of img
                              // (img is a pinned image's mapped address; k_crc_meta copies them)
    uint64_t poff;
    uint32_t *gids;
    uint64_t *sunit;
    uint32_t *lids;
    uint32_t *reg_nd;
    RegStat *rs;
    DevStats *st;
    DevStats *st_host;        // inline_meta: mapped pinned copy of the final stats
    uint64_t capacity;
    int prefetch;             // L2-prefetch each tile's next segment during the detect walk (pays at
                              // low dirty ratios, costs ~2 % when every page is rewritten)
};
void launch_fused_compare(const Launch &L, const FusedArgs &a, int blocks);

// One-launch checkpoint of a small footprint (SURVEY.md sec. 7.3 hard part 6,
// config C1): a cooperative grid detects (compare / tracked) into a page
// bitmap, meets at one grid barrier, then every CTA derives the slot of
// every dirty page from the bitmap in shared memory (no look-back): the
// CTAs gather + commit, CTA 0 writes table, ids, CRC and header.  Eligible:
// every region COMPARE or TRACKED with one page size, N <= kSmallPages,
// image >= the worst case.
constexpr uint32_t kSmallPages = 16384;
constexpr uint32_t kSmallItemsLog2 = 2;  // k_small_ckpt detect: 2^this warp work items per 4 KiB segment
struct SmallArgs {
    const DevRegion *regs;
    uint32_t R;
    uint32_t log2p;           // the context's one page size
    uint64_t N;               // pages
    uint32_t *bitmap;         // kSmallPages bits: dirty pages (zero when a launch begins; the last CTA out clears it)
    uint32_t *bar;            // [0] arrivals, [1] generation (grid barrier; persists across launches),
                              // [2] CTAs out, [4..5] ~(earliest CTA entry, ns) when timed; [0], [2], [4..5] end at 0
    uint8_t *force;
    uint8_t *img;             // image (payload at poff)
    uint64_t poff;
    uint64_t capacity;
    DevStats *st;
    DevStats *st_host;        // mapped pinned copy of the final stats (the host reads it after the kernel)
    X2N x2n;
    uint32_t timing;          // record t_ns (the kernel's own duration) in the stats
};
void launch_small_ckpt(const Launch &L, const SmallArgs &a, int blocks);
int small_blocks_per_sm();
int fused_blocks_per_sm();

// ---- detect (kernels_detect.cu) ----
void launch_detect_compare(const Launch &L, const DevRegion *regs, const uint32_t *cmp_idx,
                           const uint64_t *cmp_seg, uint32_t n_cmp, uint64_t s_lo, uint64_t s_hi,
                           const uint8_t *force, uint8_t *flags, uint8_t tag);
void launch_detect_hash(const Launch &L, const DevRegion *regs, const uint32_t *hash_idx,
                        const uint64_t *hash_grp, uint32_t n_hash, uint64_t w_lo, uint64_t w_hi,
                        uint8_t *flags, uint64_t *newhash, uint8_t tag);
// pages of P >= kBigHashPage bytes: one CTA per page (warp specialised)
constexpr uint32_t kBigHashLog2 = 16;
void launch_detect_hash_big(const Launch &L, const DevRegion *regs, const uint32_t *big_idx,
                            const uint64_t *big_pg, uint32_t n_big, uint64_t w_lo, uint64_t w_hi,
                            uint8_t *flags, uint64_t *newhash, uint8_t tag);
void launch_verify_hash(const Launch &L, const DevRegion *regs, uint32_t R, const RegStat *rs,
                        const uint64_t *hashes, const uint8_t *payload, uint64_t K, DevStats *st);

// ---- compaction, metadata, gather, scatter, CRC (kernels_image.cu) ----
void launch_compact(const Launch &L, const CompactArgs &a);
void launch_gather(const Launch &L, const GatherArgs &a, uint64_t max_units);
void launch_crc_meta(const Launch &L, const CrcArgs &a, uint64_t max_len);
void launch_crc_check(const Launch &L, const uint8_t *table, uint64_t tab, const uint8_t *tail, uint64_t tl,
                      DevStats *st, const X2N &x2n);
void launch_restore_validate(const Launch &L, const DevRegion *tregs, uint32_t R, const RegStat *rs,
                             const uint32_t *ids, const uint64_t *hashes, uint64_t K, DevStats *st);
void launch_scatter(const Launch &L, const ScatterArgs &a);

// Compressed images (kernels_zip.cu; readings Z2-Z3): per 4 KiB
// payload unit a greedy LZ77 parse coded as one fixed-Huffman DEFLATE block.
// A gather gathers the listed pages chunk by chunk into a raw staging buffer
// (k_gather, no commit), then encode -> chunk scan -> pack.  Restore offsets
// of encoded units: zblk[u / kZScanBlock] + zloc[u] (bytes from the payload).
constexpr uint32_t kZScanBlock = 2048;
constexpr uint32_t kZChunkUnits = 32768;   // at most 128 MiB of units per compressed chunk ...
constexpr uint32_t kZMinChunkUnits = 4096;  // ... at least 16 MiB (a quarter of the range's units in between)
// Encode the n units at raw (4 KiB each) into enc (same layout), sizes into zsz[0..n).
void launch_zenc(const Launch &L, const uint8_t *raw, uint64_t n, uint8_t *enc, uint16_t *zsz, const DevStats *st);
// Chunk-relative offsets zloc[0..n) of the n <= kZChunkUnits sizes; *zbase =
// the running total *zrun before the chunk; *zrun (and *zrun_host, mapped,
// nullable) advanced by the chunk's total.
void launch_zscan_chunk(const Launch &L, const uint16_t *zsz, uint64_t n, uint32_t *zloc, uint64_t *zrun,
                        uint64_t *zbase, uint64_t *zrun_host);
// Move the n encodings from stage to dst + (base ? *base : 0) + zloc[i];
// limit != 0: a unit is written only if offset + size <= limit (payload bytes that fit).
void launch_zpack(const Launch &L, const uint8_t *stage, const uint16_t *zsz, const uint32_t *zloc, uint64_t n,
                  const uint64_t *base, uint8_t *dst, uint64_t limit, const DevStats *st);
// After the last chunk: the compressed image's sizes and capacity status
// (total encoded length *zrun); zero the payload padding of img (nullable).
void launch_zfinal(const Launch &L, DevStats *st, const uint64_t *zrun, uint8_t *img, uint64_t capacity);
// Restore: validate the size table (every size <= 4096, the sizes summing to
// the header's payload length before padding) and compute zloc / zblk.
void launch_zscan(const Launch &L, const uint16_t *zsz, DevStats *st, uint32_t *zloc, uint64_t *zblk,
                  uint64_t max_units);
// Decode units [u_lo, u_lo + units) from src into dst (unit u at
// dst + (u - u_lo) * 4096; dst == nullptr: validate only).  rebase: src holds
// the payload from byte (off(u_lo) & ~3) on (k_zfetch), else from byte 0.
// An invalid unit sets st->status = CORRUPT.
void launch_zdecode(const Launch &L, const uint8_t *src, const uint16_t *zsz, const uint32_t *zloc,
                    const uint64_t *zblk, DevStats *st, uint8_t *dst, uint64_t units, uint64_t u_lo = 0,
                    int rebase = 0);
// Copy the encoded bytes of units [u_lo, u_hi) -- payload bytes
// [off(u_lo) & ~3, round_up(end, 4)) -- from src to dst (wide reads).
void launch_zfetch(const Launch &L, const uint8_t *src, const uint16_t *zsz, const uint32_t *zloc,
                   const uint64_t *zblk, uint64_t u_lo, uint64_t u_hi, uint8_t *dst);
void launch_mark_pages(const Launch &L, uint8_t *force, uint64_t n_pages, const uint32_t *pages, uint64_t n);
void launch_export_flags(const Launch &L, uint8_t *flags, const uint8_t *force, uint64_t N, uint8_t tag,
                         uint8_t *out);

// ---- synthetic inputs (synth.cu) ----
void launch_synth_fill(cudaStream_t s, uint8_t *p, uint64_t bytes, uint64_t seed, uint64_t r,
                       uint64_t word_offset);
void launch_synth_write(cudaStream_t s, uint8_t *p, uint64_t bytes, uint64_t page_size,
                        const uint32_t *pages, uint64_t n, uint64_t seed, uint64_t epoch, uint64_t r,
                        int touch, const crum_tracker *t);
void launch_synth_scrub(cudaStream_t s, uint8_t *p, uint64_t bytes);

// ---- small device helpers shared by the kernel files ----
__host__ __device__ inline uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Largest r in [0, n) with prefix[r] <= key (prefix is ascending, prefix[0] == 0).
__device__ __forceinline__ uint32_t upper_region(const uint64_t *prefix, uint32_t n, uint64_t key) {
    uint32_t lo = 0, hi = n;  // answer in [lo, hi)
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(prefix + mid) <= key) lo = mid; else hi = mid;
    }
    return lo;
}

// ---- block / warp helpers shared by the kernel files ----
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide exclusive scan of one u64 per thread; returns the exclusive
// prefix, *total = block sum.  blockDim.x must be a multiple of 32, <= 1024.
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t *total) {
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

__device__ __forceinline__ uint64_t block_sum(uint64_t v) {
    uint64_t t;
    block_excl_scan(v, &t);
    return t;
}

// Largest r with regs[r].page_base <= g.
__device__ __forceinline__ uint32_t region_of_page(const DevRegion *regs, uint32_t R, uint64_t g) {
    uint32_t lo = 0, hi = R;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (regs[mid].page_base <= g) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t page_len(const DevRegion &g, uint64_t i) {
    const uint64_t off = i << g.log2p;
    return min((uint64_t)1 << g.log2p, (uint64_t)(g.bytes - off));
}


}  // namespace crum
