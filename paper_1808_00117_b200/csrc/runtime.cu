// runtime.cu -- host runtime of libcrum.so and the C ABI of include/crum.h.
//
// Responsibilities: region registry and device
// descriptors, shadow storage (mirrors / hash tables / force bits), scratch,
// the range-pipelined gather -> D2H and the chunked H2D -> scatter paths
// (side streams, events), image header/table validation, error state.  All
// data-parallel work runs in the kernels of kernels_detect.cu and
// kernels_image.cu.
#include <cuda_runtime.h>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <cstdarg>
#include <thread>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/crum.h"
#include "crum_internal.cuh"

using namespace crum;

namespace {

thread_local std::string g_detail;

// NVTX range around an API call (header-only NVTX v3: free unless a tool such
// as ncu --nvtx is attached); ncu can then select a call's kernels by range.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

void set_detail(const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_detail = buf;
}

// --- host CRC-32 (zlib) helpers: the 60-byte header check and the device
// --- CRC kernels' x^(2^k) table.
struct CrcTables {
    uint32_t byte[256];
    X2N x2n;  // x^(2^k) mod P (reflected)
};

uint32_t gf2_mulmod_host(uint32_t a, uint32_t b) {
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

const CrcTables &crc_tables() {
    static CrcTables t = [] {
        CrcTables c{};
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t v = i;
            for (int k = 0; k < 8; ++k) v = (v >> 1) ^ (0xEDB88320u & (0u - (v & 1u)));
            c.byte[i] = v;
        }
        c.x2n.t[0] = 0x40000000u;  // x^1
        for (int k = 1; k < 32; ++k) c.x2n.t[k] = gf2_mulmod_host(c.x2n.t[k - 1], c.x2n.t[k - 1]);
        // pw[j] = x^(512 j): x^512 = x^(2^9)
        c.x2n.pw[0] = 0x80000000u;  // x^0
        for (int j = 1; j < 32; ++j) c.x2n.pw[j] = gf2_mulmod_host(c.x2n.t[9], c.x2n.pw[j - 1]);
        // lpw[j] = x^(128 j) (x^128 = x^(2^7)), wpw[w] = x^(4096 w) (x^(2^12))
        c.x2n.lpw[0] = 0x80000000u;
        for (int j = 1; j < 32; ++j) c.x2n.lpw[j] = gf2_mulmod_host(c.x2n.t[7], c.x2n.lpw[j - 1]);
        c.x2n.wpw[0] = 0x80000000u;
        for (int w = 1; w < 8; ++w) c.x2n.wpw[w] = gf2_mulmod_host(c.x2n.t[12], c.x2n.wpw[w - 1]);
        return c;
    }();
    return t;
}

uint32_t crc32_host(const uint8_t *p, size_t n) {
    const CrcTables &t = crc_tables();
    uint32_t c = 0xffffffffu;
    for (size_t i = 0; i < n; ++i) c = t.byte[(c ^ p[i]) & 0xffu] ^ (c >> 8);
    return c ^ 0xffffffffu;
}

inline uint64_t rd64(const uint8_t *p) {
    uint64_t v;
    memcpy(&v, p, 8);
    return v;
}
inline uint32_t rd32(const uint8_t *p) {
    uint32_t v;
    memcpy(&v, p, 4);
    return v;
}

// Image format v1 layout.
uint64_t payload_offset_for(uint64_t R) { return round_up(64 + 48 * R, 4096); }
uint64_t tail_bytes_for(uint64_t K, bool has_hashes) { return round_up(4 * K, 8) + (has_hashes ? 8 * K : 0); }

// The single-pass kernel's scratch, one allocation cleared by one memset per
// launch: FusedScratch (256 B) | per-region counts (4 R, to 256 B) | status
// words (8 per tile + 1).
constexpr uint64_t kFsHead = 256;
uint64_t fused_counts_bytes(uint64_t R) { return round_up(4 * R + 4, 256); }
uint64_t fused_scratch_bytes(uint64_t R, uint64_t n_tiles) {
    return kFsHead + fused_counts_bytes(R) + 8 * (n_tiles + 1);
}

struct HostRegion {
    uint32_t id;
    uint32_t mode;
    uint8_t *ptr;
    uint64_t bytes;
    uint64_t page_size;
    uint64_t n_pages;
    uint32_t log2p;
    void *shadow;  // device mirror (compare) or hash table (hash)
    uint64_t page_base;
};

// A page range of the pipelined host path, with the matching compare-segment
// and hash-group ranges of the detect kernels.
struct Range {
    uint64_t p_lo, p_hi, s_lo, s_hi, w_lo, w_hi, v_lo, v_hi;
};

constexpr uint64_t kDefaultChunk = 64ull << 20;
constexpr int kRing = 3;
constexpr int kMaxRanges = 32;
constexpr uint64_t kMinRangeBytes = 128ull << 20;
constexpr uint64_t kMaxTotalPages = 0x7fffffffull;

}  // namespace

namespace {
// Pinned, device-mapped host pool (crum_config.pinned_pool_bytes): images are
// carved from it first fit in 4 KiB granules; free extents are kept sorted by
// offset and coalesce on release.  Images may be destroyed from any thread
// (the writer thread of a persisting image joins first), so the free list has
// its own lock.
struct PinnedPool {
    uint8_t *base = nullptr;
    uint64_t bytes = 0;
    uint64_t map_bytes = 0;  // > 0: mmap + cudaHostRegister (else cudaHostAlloc)
    int numa_node = -1;
    std::mutex mu;
    std::map<uint64_t, uint64_t> free_ext;  // offset -> length
    uint64_t in_use = 0;
    uint32_t images = 0;

    uint8_t *carve(uint64_t len) {
        len = round_up(len ? len : 1, 4096);
        std::lock_guard<std::mutex> g(mu);
        for (auto it = free_ext.begin(); it != free_ext.end(); ++it) {
            if (it->second < len) continue;
            const uint64_t off = it->first, rest = it->second - len;
            free_ext.erase(it);
            if (rest) free_ext.emplace(off + len, rest);
            in_use += len;
            ++images;
            return base + off;
        }
        return nullptr;
    }
    void release(uint8_t *p, uint64_t len) {
        len = round_up(len ? len : 1, 4096);
        std::lock_guard<std::mutex> g(mu);
        in_use -= len;
        --images;
        uint64_t off = (uint64_t)(p - base);
        auto next = free_ext.lower_bound(off);
        if (next != free_ext.end() && off + len == next->first) {
            len += next->second;
            next = free_ext.erase(next);
        }
        if (next != free_ext.begin()) {
            auto prev = std::prev(next);
            if (prev->first + prev->second == off) {
                off = prev->first;
                len += prev->second;
                free_ext.erase(prev);
            }
        }
        free_ext.emplace(off, len);
    }
    uint64_t largest_free() {
        std::lock_guard<std::mutex> g(mu);
        uint64_t m = 0;
        for (const auto &e : free_ext) m = std::max(m, e.second);
        return m;
    }
};
}  // namespace

struct crum_image {
    uint8_t *host;
    uint64_t cap;
    uint64_t len;
    int device;
    uint64_t map_bytes = 0;  // > 0: mmap'ed on the device's NUMA node + cudaHostRegister'ed
    int numa_node = -1;      // node the pages were bound to (-1: cudaHostAlloc, default policy)
    PinnedPool *pool = nullptr;  // carved from the context's pool (released there on destroy)
    // asynchronous persistence (writer thread)
    std::thread writer;
    std::atomic<int> busy{0};
    int result = 0;
    std::string error;
    int sessions = 0;  // open lazy-restore sessions reading this image
};

struct crum_ctx {
    int device = 0;
    int numa_node = -1;  // images are bound to this host node (-1: default placement)
    PinnedPool *pool = nullptr;  // crum_config.pinned_pool_bytes > 0
    bool graphs_on = true;       // !CRUM_CFG_NO_GRAPH
    bool fused_cfg = false;      // CRUM_CFG_FUSED
    bool mapped_cfg = true;      // !CRUM_CFG_NO_MAPPED
    crum_restore_session *session = nullptr;  // open lazy restore (blocks other state changes)
    uint32_t last_path = 0;                   // CRUM_PATH_* bits of the last gather
    // CUDA graph of the asynchronous device gather (one cached instance)
    cudaStream_t gcap = nullptr;              // capture stream
    uint64_t graph_epoch = 1;                 // bumped by every allocation / rebuild
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        uint64_t nk = 0;                      // kernels per replay
        uint64_t epoch = 0;
        uint8_t *img = nullptr;
        uint64_t cap = 0;
        uint32_t flags = 0;
        uint64_t used = 0;                    // LRU stamp
        bool fused = false;                   // the captured sequence is the single-pass kernel
        bool small = false;                   // ... the one-launch small-footprint kernel
    };
    static constexpr int kGraphs = 4;         // e.g. two alternating images x {device, host}
    GraphEntry graphs[kGraphs];
    uint64_t graph_clock = 0;
    int sms = 148;
    uint64_t chunk = kDefaultChunk;
    std::vector<HostRegion> regs;
    std::vector<Range> ranges;
    std::vector<Range> mranges;  // the mapped-store path's ranges (halving: 1/2, 1/4, 1/4)
    std::vector<Range> zranges;  // compressed pinned gathers: as ranges, from 64 MiB
    Range all{};
    uint32_t next_id = 1;
    uint64_t N = 0, F = 0, max_units = 0;
    bool poisoned = false;
    uint64_t launches = 0;
    uint8_t tag = 0;

    // device descriptors (rebuilt on register / unregister)
    DevRegion *d_regs = nullptr;
    uint32_t *d_cmp_idx = nullptr;
    uint64_t *d_cmp_seg = nullptr;
    uint32_t n_cmp = 0;
    uint32_t *d_hash_idx = nullptr;
    uint64_t *d_hash_grp = nullptr;
    uint32_t n_hash = 0;
    uint32_t *d_big_idx = nullptr;   // hash regions with P >= 64 KiB (CTA per page)
    uint64_t *d_big_pg = nullptr;
    uint32_t n_big = 0;
    bool any_hash = false;

    // single-pass (fused) checkpoint: all regions COMPARE with P <= 64 KiB
    bool fused_ok = false;
    uint64_t *d_tile_base = nullptr;
    uint64_t n_tiles = 0;
    uint32_t *d_small = nullptr;   // one-launch small path: dirty bitmap | grid barrier words
    bool small_ok = false;         // every region COMPARE/TRACKED, one page size, N <= kSmallPages, F small
    uint32_t small_log2p = 12;
    int small_bps = 1;
    uint64_t *d_status = nullptr;  // single-pass scratch: FusedScratch | per-region counts | status words
    uint32_t fused_tile_min = 15;
    int fused_bps = 1;
    bool last_fused = false;

    // per-page arrays (padded to kPagesPerCompactBlock)
    uint64_t page_cap = 0;
    uint8_t *d_force = nullptr;
    uint8_t *d_flags = nullptr;
    uint64_t *d_newhash = nullptr;
    uint32_t *d_gids = nullptr;
    uint64_t *d_sunit = nullptr;
    uint32_t *d_u2s = nullptr;     // payload unit -> slot (written by compaction)
    uint64_t u2s_cap = 0;
    uint32_t *d_lids = nullptr;
    uint64_t *d_lhash = nullptr;
    uint64_t *d_blk_units = nullptr;
    uint8_t *d_dbg = nullptr;

    uint32_t *d_reg_nd = nullptr;
    RegStat *d_rs = nullptr;
    uint64_t rs_cap = 0;
    DevRegion *d_tregs = nullptr;  // restore: descriptors built from an image table
    uint64_t tregs_cap = 0;
    RangeTotals *d_rb = nullptr;   // kMaxRanges + 1
    RangeTotals *h_rb = nullptr;   // pinned, mapped mirror
    uint32_t *d_done = nullptr;    // [0] compaction, [1] crc
    // compressed images: per-unit encoded sizes, local offsets, block offsets
    uint16_t *d_zsz = nullptr;
    uint32_t *d_zloc = nullptr;
    uint64_t *d_zblk = nullptr;
    uint64_t z_cap = 0;            // units the three arrays hold
    uint64_t *d_zrun = nullptr;    // running encoded length of a compressed gather
    uint8_t *d_zstage = nullptr;   // one chunk of encoded units (raw layout, kZChunkUnits x 4 KiB)
    uint8_t *d_zraw = nullptr;     // one chunk of gathered (not yet encoded) units
    uint64_t *h_zrun = nullptr;    // pinned, mapped: running length after each chunk ([0] = 0)
    uint64_t *dh_zrun = nullptr;   // device address of h_zrun
    uint64_t *d_zbase = nullptr;   // per chunk: the running encoded length before it
    // restore staging kept across calls (grow-only): decoded / verified payload, encoded payload
    uint8_t *d_rtmp = nullptr;
    uint64_t rtmp_cap = 0;
    uint8_t *d_renc = nullptr;
    uint64_t renc_cap = 0;
    DevStats *d_st = nullptr;
    DevStats *h_st = nullptr;      // pinned, mapped
    DevStats *dh_st = nullptr;     // its device address
    RangeTotals *dh_rb = nullptr;  // device address of h_rb (mapped)

    uint8_t *d_meta = nullptr;     // host path: image head [0, poff) then the tail
    uint64_t meta_cap = 0;
    uint8_t *d_ring[kRing] = {nullptr, nullptr, nullptr};
    uint64_t ring_cap = 0;

    cudaStream_t copy = nullptr;    // D2H / H2D
    cudaStream_t gstream = nullptr; // gathers of the pipelined host path
    cudaStream_t aux = nullptr;     // device path: metadata CRC beside the gather
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_gather[kRing];
    cudaEvent_t ev_copy[kRing];
    cudaEvent_t ev_range[kMaxRanges];
    cudaEvent_t ev_t[6];
    cudaEvent_t ev_meta;
    // CRUM_CFG_TRACE: per-range timing events of the host path, printed to stderr
    bool trace = false;
    uint64_t gathers_since_rebuild = 0;  // pinned gathers since the registry changed
    cudaEvent_t ev_trace[3 * kMaxRanges] = {};
    // CRUM_CFG_TIMING and the most recent call (crum_last_report)
    bool timing_cfg = false;
    int last_kind = 0;      // 0 none, 1 sync, 2 device gather, 3 host gather, 4 restore
    bool last_small = false;  // with kLastDevFused: the one-launch small kernel (two events)
    bool last_timed = false;
    cudaEvent_t ev_done = nullptr;
};

namespace {

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_detail("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
            c->poisoned = true;                                                               \
            return CRUM_E_CUDA;                                                               \
        }                                                                                     \
    } while (0)

#define CK_LAUNCH()                                                                           \
    do {                                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess) {                                                              \
            set_detail("kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
            c->poisoned = true;                                                               \
            return CRUM_E_CUDA;                                                               \
        }                                                                                     \
    } while (0)

#define ENTER(ctx)                                                                            \
    crum_ctx *c = (ctx);                                                                      \
    if (!c) {                                                                                 \
        set_detail("null context");                                                           \
        return CRUM_E_INVAL;                                                                  \
    }                                                                                         \
    if (c->poisoned) {                                                                        \
        set_detail("context poisoned by an earlier CUDA error");                              \
        return CRUM_E_CUDA;                                                                   \
    }                                                                                         \
    CK(cudaSetDevice(c->device))

#define NOT_IN_SESSION(c)                                                                     \
    if ((c)->session) {                                                                       \
        set_detail("a lazy restore session is open (crum_restore_end first)");               \
        return CRUM_E_BUSY;                                                                   \
    }

Launch launch_of(crum_ctx *c, cudaStream_t s) { return Launch{s, c->sms, &c->launches}; }

uint64_t pad_pages(uint64_t n) { return round_up(n ? n : 1, kPagesPerCompactBlock); }

template <typename T>
int dev_alloc(crum_ctx *c, T **p, uint64_t bytes) {
    ++c->graph_epoch;  // a captured graph may hold the pointer this replaces
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_detail("cudaMalloc(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
        return CRUM_E_NOMEM;
    }
    *p = static_cast<T *>(q);
    return CRUM_OK;
}

template <typename T>
void dev_free(T *&p) {
    if (p) cudaFree(p);
    p = nullptr;
}

int upload(crum_ctx *c, void *dst, const void *src, uint64_t bytes) {
    if (bytes) CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return CRUM_OK;
}

// Compare segments / hash groups of the pages before global page p.
uint64_t seg_at(const crum_ctx *c, uint64_t p) {
    uint64_t s = 0;
    for (const HostRegion &h : c->regs) {
        if (h.mode != kModeCompare) continue;
        if (p >= h.page_base + h.n_pages) s += (h.bytes + kSegBytes - 1) / kSegBytes;
        else if (p > h.page_base) s += (p - h.page_base) << (h.log2p - kSegLog2);
    }
    return s;
}
uint64_t grp_at(const crum_ctx *c, uint64_t p, bool ceil) {
    uint64_t w = 0;
    for (const HostRegion &h : c->regs) {
        if (h.mode != kModeHash || h.log2p >= kBigHashLog2) continue;
        const uint64_t k = p >= h.page_base + h.n_pages ? h.n_pages : (p > h.page_base ? p - h.page_base : 0);
        w += h.log2p == kSegLog2 ? (ceil ? (k + 1) / 2 : k / 2) : k;
    }
    return w;
}

uint64_t big_at(const crum_ctx *c, uint64_t p) {
    uint64_t w = 0;
    for (const HostRegion &h : c->regs) {
        if (h.mode != kModeHash || h.log2p < kBigHashLog2) continue;
        w += p >= h.page_base + h.n_pages ? h.n_pages : (p > h.page_base ? p - h.page_base : 0);
    }
    return w;
}

Range make_range(const crum_ctx *c, uint64_t lo, uint64_t hi) {
    return Range{lo, hi, seg_at(c, lo), seg_at(c, hi), grp_at(c, lo, false), grp_at(c, hi, true), big_at(c, lo),
                 big_at(c, hi)};
}

// Rebuild device descriptors and per-page arrays for the registry `regs`
// (the live one after a register / unregister).  Transactional: every new
// buffer is allocated and filled into a temporary first; only when all of
// that succeeded are the old buffers freed and c->regs replaced, so a
// CRUM_E_NOMEM leaves the context exactly as it was (crum.h conventions).
// old_force_base[r]: page base of region r's force bits in the CURRENT force
// array, or UINT64_MAX for a new region (all force-dirty).
int rebuild(crum_ctx *c, std::vector<HostRegion> regs, const std::vector<uint64_t> &old_force_base) {
    const uint32_t R = (uint32_t)regs.size();
    std::vector<DevRegion> dr(R);
    std::vector<uint32_t> cmp_idx, hash_idx, big_idx;
    std::vector<uint64_t> cmp_seg{0}, hash_grp{0}, big_pg{0};
    uint64_t N = 0, F = 0, units = 0;
    bool any_hash = false;
    for (uint32_t r = 0; r < R; ++r) {
        HostRegion &h = regs[r];
        h.page_base = N;
        DevRegion &d = dr[r];
        d.base = h.ptr;
        d.mirror = h.mode == kModeCompare ? static_cast<uint8_t *>(h.shadow) : nullptr;
        d.table = h.mode == kModeHash ? static_cast<uint64_t *>(h.shadow) : nullptr;
        d.bytes = h.bytes;
        d.page_base = N;
        d.n_pages = h.n_pages;
        d.log2p = h.log2p;
        d.mode = h.mode;
        d.id = h.id;
        d.aligned32 = (reinterpret_cast<uintptr_t>(h.ptr) & 31) == 0;
        if (h.mode == kModeCompare) {
            cmp_idx.push_back(r);
            cmp_seg.push_back(cmp_seg.back() + (h.bytes + kSegBytes - 1) / kSegBytes);
        } else if (h.mode == kModeHash) {
            any_hash = true;
            if (h.log2p >= kBigHashLog2) {
                big_idx.push_back(r);
                big_pg.push_back(big_pg.back() + h.n_pages);
            } else {
                hash_idx.push_back(r);
                hash_grp.push_back(hash_grp.back() + (h.log2p == 12 ? (h.n_pages + 1) / 2 : h.n_pages));
            }
        }
        N += h.n_pages;
        F += h.bytes;
        units += h.n_pages << (h.log2p - kSegLog2);
    }
    // single-pass eligibility and its tile map
    bool fused_ok = R > 0 && (units >> 27) == 0;
    // small footprints: one page per tile (every warp's tile is one memory
    // round trip); large ones: >= 32 KiB per tile
    const uint32_t tile_min = F <= kFusedSmallBytes ? kSegLog2 : kFusedMinTileLog2;
    std::vector<uint64_t> tb{0};
    for (const HostRegion &h : regs) {
        fused_ok = fused_ok && h.mode == kModeCompare && h.log2p <= kFusedMaxLog2P;
        const uint32_t tl = std::max(h.log2p, tile_min);
        tb.push_back(tb.back() + ((h.bytes + (1ull << tl) - 1) >> tl));
    }
    const uint64_t cap = pad_pages(N);
    const bool grow_pages = cap > c->page_cap;
    const bool grow_u2s = units + 1 > c->u2s_cap;
    const bool grow_rs = R + 1 > c->rs_cap;
    const uint64_t meta_max = payload_offset_for(R) + tail_bytes_for(N, true) + 4096;
    const bool grow_meta = meta_max > c->meta_cap;

    // ---- phase 1: allocate every new buffer into temporaries ----
    struct Tmp {
        uint8_t *force = nullptr, *flags = nullptr, *dbg = nullptr, *meta = nullptr;
        uint64_t *newhash = nullptr, *sunit = nullptr, *lhash = nullptr, *blk_units = nullptr;
        uint32_t *gids = nullptr, *lids = nullptr, *u2s = nullptr, *reg_nd = nullptr;
        DevRegion *regs = nullptr;
        uint32_t *cmp_idx = nullptr, *hash_idx = nullptr, *big_idx = nullptr;
        uint64_t *cmp_seg = nullptr, *hash_grp = nullptr, *big_pg = nullptr, *tile_base = nullptr, *status = nullptr;
        RegStat *rs = nullptr;
        void free_all() {
            dev_free(force); dev_free(flags); dev_free(dbg); dev_free(meta); dev_free(newhash); dev_free(sunit);
            dev_free(lhash); dev_free(blk_units); dev_free(gids); dev_free(lids); dev_free(u2s); dev_free(reg_nd);
            dev_free(regs); dev_free(cmp_idx); dev_free(hash_idx); dev_free(big_idx); dev_free(cmp_seg);
            dev_free(hash_grp); dev_free(big_pg); dev_free(tile_base); dev_free(status); dev_free(rs);
        }
    } t;
    const uint64_t nblk = cap / kPagesPerCompactBlock + 1;
    int st = CRUM_OK;
    auto alloc_all = [&]() -> int {
        int e;
        if ((e = dev_alloc(c, &t.force, cap))) return e;
        if (grow_pages &&
            ((e = dev_alloc(c, &t.flags, cap)) || (e = dev_alloc(c, &t.newhash, cap * 8)) ||
             (e = dev_alloc(c, &t.gids, cap * 4)) || (e = dev_alloc(c, &t.sunit, cap * 8)) ||
             (e = dev_alloc(c, &t.lids, cap * 4 + 8)) || (e = dev_alloc(c, &t.lhash, cap * 8)) ||
             (e = dev_alloc(c, &t.blk_units, nblk * 8)) || (e = dev_alloc(c, &t.dbg, cap))))
            return e;
        if ((e = dev_alloc(c, &t.regs, sizeof(DevRegion) * R)) || (e = dev_alloc(c, &t.cmp_idx, 4 * cmp_idx.size())) ||
            (e = dev_alloc(c, &t.cmp_seg, 8 * cmp_seg.size())) || (e = dev_alloc(c, &t.hash_idx, 4 * hash_idx.size())) ||
            (e = dev_alloc(c, &t.hash_grp, 8 * hash_grp.size())) || (e = dev_alloc(c, &t.reg_nd, 4 * R + 4)) ||
            (e = dev_alloc(c, &t.big_idx, 4 * big_idx.size())) || (e = dev_alloc(c, &t.big_pg, 8 * big_pg.size())))
            return e;
        if (grow_u2s && (e = dev_alloc(c, &t.u2s, 4 * (units + 1)))) return e;
        if (fused_ok && ((e = dev_alloc(c, &t.tile_base, 8 * tb.size())) ||
                         (e = dev_alloc(c, &t.status, fused_scratch_bytes(R, tb.back())))))
            return e;
        if (grow_rs && (e = dev_alloc(c, &t.rs, sizeof(RegStat) * (R + 1)))) return e;
        if (grow_meta && (e = dev_alloc(c, &t.meta, meta_max))) return e;
        return CRUM_OK;
    };
    if ((st = alloc_all())) {
        t.free_all();
        return st;
    }
    // ---- phase 2: fill them (CUDA errors here poison the context) ----
    auto fill_all = [&]() -> int {
        CK(cudaMemset(t.force, 0, cap));
        // carry the force bits of surviving regions over, new regions all
        // force-dirty; consecutive regions that keep their relative layout
        // (every region of an append, the two sides of an unregister) move
        // as one copy / one memset, so registering R regions one by one
        // costs O(R) calls, not O(R^2)
        uint64_t run_dst = 0, run_src = UINT64_MAX, run_len = 0;
        bool run_new = false;
        auto flush = [&]() -> int {
            if (run_len) {
                if (run_new) CK(cudaMemset(t.force + run_dst, 1, run_len));
                else CK(cudaMemcpy(t.force + run_dst, c->d_force + run_src, run_len, cudaMemcpyDeviceToDevice));
            }
            run_len = 0;
            return CRUM_OK;
        };
        for (uint32_t r = 0; r < R; ++r) {
            const uint64_t ob = old_force_base[r];
            const bool is_new = ob == UINT64_MAX;
            const uint64_t nb = dr[r].page_base;
            const bool extends = run_len && is_new == run_new && run_dst + run_len == nb &&
                                 (is_new || run_src + run_len == ob);
            if (!extends) {
                int e = flush();
                if (e) return e;
                run_dst = nb;
                run_src = ob;
                run_new = is_new;
            }
            run_len += dr[r].n_pages;
        }
        {
            int e = flush();
            if (e) return e;
        }
        int e;
        if ((e = upload(c, t.regs, dr.data(), sizeof(DevRegion) * R)) ||
            (e = upload(c, t.cmp_idx, cmp_idx.data(), 4 * cmp_idx.size())) ||
            (e = upload(c, t.cmp_seg, cmp_seg.data(), 8 * cmp_seg.size())) ||
            (e = upload(c, t.hash_idx, hash_idx.data(), 4 * hash_idx.size())) ||
            (e = upload(c, t.hash_grp, hash_grp.data(), 8 * hash_grp.size())) ||
            (e = upload(c, t.big_idx, big_idx.data(), 4 * big_idx.size())) ||
            (e = upload(c, t.big_pg, big_pg.data(), 8 * big_pg.size())))
            return e;
        if (fused_ok) {
            if ((e = upload(c, t.tile_base, tb.data(), 8 * tb.size()))) return e;
            CK(cudaMemset(t.status, 0, fused_scratch_bytes(R, tb.back())));
        }
        return CRUM_OK;
    };
    if ((st = fill_all())) {
        t.free_all();
        return st;
    }
    // ---- phase 3: commit (frees cannot fail) ----
    auto swap_in = [](auto *&dst, auto *&src) {
        dev_free(dst);
        dst = src;
        src = nullptr;
    };
    swap_in(c->d_force, t.force);
    if (grow_pages) {
        swap_in(c->d_flags, t.flags);
        swap_in(c->d_newhash, t.newhash);
        swap_in(c->d_gids, t.gids);
        swap_in(c->d_sunit, t.sunit);
        swap_in(c->d_lids, t.lids);
        swap_in(c->d_lhash, t.lhash);
        swap_in(c->d_blk_units, t.blk_units);
        swap_in(c->d_dbg, t.dbg);
        c->page_cap = cap;
    }
    swap_in(c->d_regs, t.regs);
    swap_in(c->d_cmp_idx, t.cmp_idx);
    swap_in(c->d_cmp_seg, t.cmp_seg);
    swap_in(c->d_hash_idx, t.hash_idx);
    swap_in(c->d_hash_grp, t.hash_grp);
    swap_in(c->d_big_idx, t.big_idx);
    swap_in(c->d_big_pg, t.big_pg);
    swap_in(c->d_reg_nd, t.reg_nd);
    if (grow_u2s) {
        swap_in(c->d_u2s, t.u2s);
        c->u2s_cap = units + 1;
    }
    swap_in(c->d_tile_base, t.tile_base);
    swap_in(c->d_status, t.status);
    c->fused_ok = fused_ok;
    c->n_tiles = fused_ok ? tb.back() : 0;
    c->fused_tile_min = tile_min;
    {
        bool ok = R > 0 && N <= kSmallPages && F <= kFusedSmallBytes;
        for (const HostRegion &h : regs)
            ok = ok && (h.mode == kModeCompare || h.mode == kModeTracked) && h.log2p == regs[0].log2p;
        c->small_ok = ok;
        c->small_log2p = R ? regs[0].log2p : 12;
    }
    if (grow_rs) {
        swap_in(c->d_rs, t.rs);
        c->rs_cap = R + 1;
    }
    if (grow_meta) {
        swap_in(c->d_meta, t.meta);
        c->meta_cap = meta_max;
    }
    // detect marks are zero between calls; single-pass compaction's look-back
    // status words start (and are left) zero
    CK(cudaMemset(c->d_flags, 0, c->page_cap));
    CK(cudaMemset(c->d_blk_units, 0, 8 * (c->page_cap / kPagesPerCompactBlock + 1)));
    c->tag = 0;
    c->regs = std::move(regs);
    c->n_cmp = (uint32_t)cmp_idx.size();
    c->n_hash = (uint32_t)hash_idx.size();
    c->n_big = (uint32_t)big_idx.size();
    c->any_hash = any_hash;
    c->N = N;
    c->F = F;
    c->max_units = units;
    // page ranges of the pipelined host path, boundaries on multiples of 16
    // pages: the first ranges are small (the host link starts early), then
    // they double up to ~F/8 (>= 128 MiB) each
    c->all = make_range(c, 0, N);
    c->ranges.clear();
    c->gathers_since_rebuild = 0;  // every page of a new region is force-dirty
    // A range holding large-page hash pages keeps at least one such page per
    // SM: their per-page scramble chain is serial, so a 16 MiB range of 2 MiB
    // pages (8 pages) would run on 8 CTAs.  (One page per CTA slot, 3 per SM,
    // delayed the first copy more than it saved: C2 hash 2 MiB e2e 482 vs 502.)
    const uint64_t min_big = (uint64_t)std::max(c->sms, 1);
    const uint64_t target_max = std::max(kMinRangeBytes, F / 8);
    auto build_ranges = [&](std::vector<Range> &out, uint64_t target) {
        out.clear();
        uint64_t lo = 0, acc = 0, nbig = 0;
        for (uint32_t r = 0; r < R; ++r) {
            const HostRegion &h = c->regs[r];
            const bool big_hash = h.mode == kModeHash && h.log2p >= 16;
            for (uint64_t i = 0; i < h.n_pages; ++i) {
                const uint64_t g = h.page_base + i;
                if (acc >= target && (nbig == 0 || nbig >= min_big) && g % 16 == 0 &&
                    (int)out.size() < kMaxRanges - 1) {
                    out.push_back(make_range(c, lo, g));
                    lo = g;
                    acc = 0;
                    nbig = 0;
                    target = std::min(target_max, 2 * target);
                }
                // whole pages at a time is fine for large regions; skip ahead in big steps
                const uint64_t step = std::min<uint64_t>(h.n_pages - i, 16 - (g % 16));
                acc += step * h.page_size;
                if (big_hash) nbig += step;
                i += step - 1;
            }
        }
        out.push_back(make_range(c, lo, N));
    };
    build_ranges(c->ranges, std::max<uint64_t>(16ull << 20, F / 128));
    // Compressed gathers start from 64 MiB ranges: a chunk's way to the link
    // (detect, compact, host wake, gather, encode ~30 us, scan, pack, host
    // wake) is ~100 us, which the first ranges' short copies did not cover
    build_ranges(c->zranges, std::max<uint64_t>(64ull << 20, F / 32));
    uint64_t lo = 0;
    // The mapped-store path's ranges: the stores of range c overlap the
    // detection of range c + 1 and every boundary costs a kernel drain, so a
    // few ranges of decreasing size -- the first half, a quarter, the rest --
    // cut on multiples of 16 pages.  Not with large-page hash pages: their
    // serial chains want every page of the footprint in one launch (C2 hash
    // 2 MiB at 1 %: two ranges of 256 pages 0.465 ms, one range 0.435 ms).
    c->mranges.clear();
    if (big_at(c, N) == 0)
        for (const uint64_t want : {N / 2, (3 * N) / 4}) {
            const uint64_t g = want / 16 * 16;
            if (g <= lo || g >= N) continue;
            c->mranges.push_back(make_range(c, lo, g));
            lo = g;
        }
    c->mranges.push_back(make_range(c, lo, N));
    return CRUM_OK;
}

// Grow-only device buffer.
int grow(crum_ctx *c, uint8_t **p, uint64_t *cap, uint64_t bytes) {
    if (*cap >= bytes && *p) return CRUM_OK;
    dev_free(*p);
    *cap = 0;
    int st = dev_alloc(c, p, bytes);
    if (st) return st;
    *cap = bytes;
    return CRUM_OK;
}

// Scratch of compressed gathers / restores for `units` 4 KiB units.
int ensure_z(crum_ctx *c, uint64_t units) {
    if (c->z_cap >= units && c->d_zsz) return CRUM_OK;
    dev_free(c->d_zsz);
    dev_free(c->d_zloc);
    dev_free(c->d_zblk);
    if (c->h_zrun) cudaFreeHost(c->h_zrun);
    c->h_zrun = c->dh_zrun = nullptr;
    c->z_cap = 0;
    int st;
    if ((st = dev_alloc(c, &c->d_zsz, 2 * (units + 8))) || (st = dev_alloc(c, &c->d_zloc, 4 * (units + 8))) ||
        (st = dev_alloc(c, &c->d_zblk, 8 * (units / kZScanBlock + 2))))
        return st;
    if (!c->d_zrun && (st = dev_alloc(c, &c->d_zrun, 8))) return st;
    const uint64_t nrun = units / kZMinChunkUnits + kMaxRanges + 2;  // chunks: per range, then by size
    dev_free(c->d_zbase);
    if ((st = dev_alloc(c, &c->d_zbase, 8 * nrun))) return st;  // each chunk's base offset
    // + slack: the pack kernel's funnel shift reads one word past a unit
    if (!c->d_zstage && (st = dev_alloc(c, &c->d_zstage, ((uint64_t)kZChunkUnits << kSegLog2) + 256))) return st;
    if (!c->d_zraw && (st = dev_alloc(c, &c->d_zraw, (uint64_t)kZChunkUnits << kSegLog2))) return st;
    void *dp = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void **>(&c->h_zrun), 8 * nrun, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&dp, c->h_zrun, 0) != cudaSuccess) {
        cudaGetLastError();
        if (c->h_zrun) cudaFreeHost(c->h_zrun);
        c->h_zrun = nullptr;
        set_detail("cudaHostAlloc of the compressed-chunk table failed");
        return CRUM_E_NOMEM;
    }
    c->dh_zrun = static_cast<uint64_t *>(dp);
    c->z_cap = units;
    return CRUM_OK;
}

// A pinned gather whose previous payload was at most this runs as one range.
constexpr uint64_t kOneRangePayload = 16ull << 20;
// Mapped-store gathers (gather_mapped, previous payload <= kOneRangePayload,
// or <= kMappedFusedPayload in a compare-only context): above
// kMappedSerialPayload a compare-only context runs the single pass; otherwise
// above kMappedOneRange the kernel sequence runs in c->mranges (stores
// overlapping the next range's detection), at most it in one range.
constexpr uint64_t kMappedSerialPayload = 2ull << 20;
constexpr uint64_t kMappedOneRange = 1ull << 20;
// (C2, profiles/r02/mapped/fused_32m_ab/: d = 2 % 0.57 ms mapped single pass vs
// 0.72 ms ring; 5 % 1.17 vs 1.14; 7 % 1.49 vs 1.50)
constexpr uint64_t kMappedFusedPayload = 32ull << 20;

// Host images whose worst case is at most this (and at most one pipeline
// chunk) take the zero-copy path.
constexpr uint64_t kSmallImage = 16ull << 20;

int ensure_ring(crum_ctx *c, uint64_t min_bytes = 0) {
    const uint64_t want = std::max(c->chunk, min_bytes);
    if (c->ring_cap >= want) return CRUM_OK;
    for (int i = 0; i < kRing; ++i) dev_free(c->d_ring[i]);
    c->ring_cap = 0;
    for (int i = 0; i < kRing; ++i) {
        int st = dev_alloc(c, &c->d_ring[i], want);
        if (st) return st;
    }
    c->ring_cap = want;
    return CRUM_OK;
}

HostRegion *find_region(crum_ctx *c, uint32_t id, uint32_t *index = nullptr) {
    for (uint32_t r = 0; r < c->regs.size(); ++r)
        if (c->regs[r].id == id) {
            if (index) *index = r;
            return &c->regs[r];
        }
    return nullptr;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0.f;
    }
    return ms;
}

// Detect marks changed pages with kFlagTag; compaction (and the debug export)
// clear the marks they consume, so the flags are zero between calls.
constexpr uint8_t kFlagTag = 1;

void enqueue_detect(crum_ctx *c, cudaStream_t s, const Range &rg, bool full) {
    Launch L = launch_of(c, s);
    if (!full)
        launch_detect_compare(L, c->d_regs, c->d_cmp_idx, c->d_cmp_seg, c->n_cmp, rg.s_lo, rg.s_hi, c->d_force,
                              c->d_flags, kFlagTag);
    launch_detect_hash_big(L, c->d_regs, c->d_big_idx, c->d_big_pg, c->n_big, rg.v_lo, rg.v_hi, c->d_flags,
                           c->d_newhash, kFlagTag);
    launch_detect_hash(L, c->d_regs, c->d_hash_idx, c->d_hash_grp, c->n_hash, rg.w_lo, rg.w_hi, c->d_flags,
                       c->d_newhash, kFlagTag);
}

CompactArgs compact_args(crum_ctx *c, const Range &rg, uint32_t ci, bool first, bool final, bool full,
                         uint64_t capacity, uint8_t *head) {
    CompactArgs a{};
    a.flags = c->d_flags;
    a.force = c->d_force;
    a.regs = c->d_regs;
    a.newhash = c->d_newhash;
    a.p_lo = rg.p_lo;
    a.p_hi = rg.p_hi;
    a.R = (uint32_t)c->regs.size();
    a.tag = kFlagTag;
    a.full = full ? 1 : 0;
    a.has_hashes = c->any_hash ? 1 : 0;
    a.first_range = first ? 1 : 0;
    a.final_range = final ? 1 : 0;
    a.c = ci;
    a.blk_units = c->d_blk_units;
    a.gids = c->d_gids;
    a.sunit = c->d_sunit;
    a.u2s = c->d_u2s;
    a.lids = c->d_lids;
    a.lhash = c->d_lhash;
    a.reg_nd = c->d_reg_nd;
    a.rb = c->d_rb;
    a.rb_host = c->dh_rb;
    a.done = c->d_done;
    a.rs = c->d_rs;
    a.st = c->d_st;
    a.capacity = capacity;
    a.head = head;
    return a;
}

// Compaction of one range (an empty range still runs one block, whose "last
// block" step advances the running totals and finalises).
void enqueue_compact(crum_ctx *c, cudaStream_t s, const CompactArgs &a) { launch_compact(launch_of(c, s), a); }

CrcArgs crc_args(crum_ctx *c, uint8_t *head, uint8_t *tail) {
    CrcArgs a{};
    a.head = head;
    a.tail = tail;
    a.lids = c->d_lids;
    a.lhash = c->d_lhash;
    a.gids = c->d_gids;
    a.st = c->d_st;
    a.done = c->d_done + 1;
    a.st_host = c->dh_st;
    a.x2n = crc_tables().x2n;
    a.zsz = c->d_zsz;
    return a;
}

GatherArgs gather_args(crum_ctx *c, uint32_t ci, uint8_t *dst, uint64_t dst_unit0, bool add_poff, uint64_t u_lo,
                       uint64_t u_hi) {
    GatherArgs a{};
    a.regs = c->d_regs;
    a.R = (uint32_t)c->regs.size();
    a.add_poff = add_poff ? 1 : 0;
    a.gids = c->d_gids;
    a.sunit = c->d_sunit;
    a.u2s = c->d_u2s;
    a.newhash = c->d_newhash;
    a.rb = c->d_rb + ci;
    a.st = c->d_st;
    a.dst = dst;
    a.dst_unit0 = dst_unit0;
    a.force = c->d_force;
    a.u_lo = u_lo;
    a.u_hi = u_hi;
    return a;
}

uint64_t crc_max_len(const crum_ctx *c) { return 48ull * c->regs.size() + 12 * c->N + 2 * c->max_units + 16; }

void fill_report(crum_ctx *c, const DevStats &h, crum_report *rep) {
    rep->scanned_pages = c->N;
    rep->scanned_bytes = c->F;
    rep->dirty_pages = h.K;
    rep->dirty_bytes = h.dirty_bytes;
    rep->dirty_runs = h.dirty_runs;
    rep->image_bytes = h.image_bytes;
}

enum { kLastNone = 0, kLastSync = 1, kLastDevGather = 2, kLastHostGather = 3, kLastRestore = 4, kLastDevFused = 5 };

// Phase times of the most recent call from its events (see each call for
// which events delimit which phase).
void fill_times(crum_ctx *c, const DevStats &h, crum_report *rep) {
    cudaEvent_t *e = c->ev_t;
    switch (c->last_kind) {
        case kLastSync:
            rep->t_detect_ms = ev_ms(e[0], e[1]);
            rep->t_compact_ms = ev_ms(e[1], e[2]);
            rep->t_gather_ms = ev_ms(e[2], e[4]);
            rep->t_total_ms = ev_ms(e[0], e[4]);
            break;
        case kLastDevFused:
            if (c->last_small) {  // one kernel, timed by itself (first CTA in -> last CTA out)
                rep->t_detect_ms = rep->t_total_ms = h.t_ns * 1e-6;
                rep->path = CRUM_PATH_FUSED | CRUM_PATH_SMALL;
                break;
            }
            rep->t_detect_ms = ev_ms(e[0], e[1]);   // detect + compact + gather (one kernel)
            rep->t_compact_ms = ev_ms(e[1], e[4]);  // metadata CRC + header
            rep->t_total_ms = ev_ms(e[0], e[4]);
            rep->path = CRUM_PATH_FUSED;
            break;
        case kLastDevGather:
            rep->t_detect_ms = ev_ms(e[0], e[1]);
            rep->t_compact_ms = ev_ms(e[1], e[2]) + ev_ms(e[3], e[4]);
            rep->t_gather_ms = ev_ms(e[2], e[3]);
            rep->t_total_ms = ev_ms(e[0], e[4]);
            break;
        case kLastHostGather:
            rep->t_detect_ms = ev_ms(e[0], e[1]);
            rep->t_gather_ms = ev_ms(e[0], e[3]);
            rep->t_copy_ms = ev_ms(e[4], e[5]);
            rep->t_total_ms = ev_ms(e[0], e[5]);
            break;
        case kLastRestore:
            rep->t_compact_ms = ev_ms(e[0], e[1]);
            rep->t_gather_ms = ev_ms(e[1], e[3]);
            rep->t_copy_ms = ev_ms(e[4], e[5]);
            rep->t_total_ms = ev_ms(e[0], e[3]);
            break;
        default:
            break;
    }
    rep->path |= c->last_path;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char *crum_status_string(int s) {
    switch (s) {
        case CRUM_OK: return "ok";
        case CRUM_E_INVAL: return "invalid argument";
        case CRUM_E_OVERLAP: return "region overlaps a live region";
        case CRUM_E_NOREGION: return "unknown region id";
        case CRUM_E_RANGE: return "range outside the region";
        case CRUM_E_NOMEM: return "out of device or pinned memory";
        case CRUM_E_CAPACITY: return "image buffer too small";
        case CRUM_E_CORRUPT: return "corrupt image";
        case CRUM_E_MISMATCH: return "image does not match the registered regions";
        case CRUM_E_BUSY: return "busy";
        case CRUM_E_DEVICE: return "pointer or device not usable";
        case CRUM_E_CUDA: return "CUDA error";
        case CRUM_E_IO: return "file I/O error";
        default: return "unknown status";
    }
}

const char *crum_last_error_detail(void) { return g_detail.c_str(); }

namespace {

// NUMA node of a CUDA device's PCIe function (sysfs), or -1 when unknown or
// when the host has a single node (then placement is moot).
int device_numa_node(int device) {
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    for (char *q = bus; *q; ++q) *q = (char)tolower(*q);
    char path[128];
    int node = -1;
    for (const char *fmt : {"/sys/bus/pci/devices/%s/numa_node", "/sys/bus/pci/devices/0000%s/numa_node"}) {
        snprintf(path, sizeof path, fmt, bus + (strlen(bus) > 12 ? 4 : 0));
        if (FILE *f = fopen(path, "r")) {
            if (fscanf(f, "%d", &node) != 1) node = -1;
            fclose(f);
            break;
        }
    }
    if (node < 0) return -1;
    int nodes = 0;
    for (int n = 0; n < 64; ++n) {
        snprintf(path, sizeof path, "/sys/devices/system/node/node%d", n);
        struct stat sb;
        if (stat(path, &sb) == 0) ++nodes;
    }
    return nodes > 1 ? node : -1;
}

// Pinned, device-mapped host memory whose pages live on `node`: anonymous
// mmap, mbind(MPOL_PREFERRED) before the first touch, then cudaHostRegister
// (which faults the pages in under that policy and pins them).  *bound tells
// whether mbind took effect (a sandbox without CAP_SYS_NICE may refuse it;
// the memory is still pinned and mapped).  Returns nullptr if the mapping or
// the registration fails (the caller falls back to cudaHostAlloc).
uint8_t *numa_pinned_alloc(uint64_t bytes, int node, uint64_t *map_bytes, bool *bound) {
    const uint64_t pg = (uint64_t)sysconf(_SC_PAGESIZE);
    const uint64_t len = (bytes + pg - 1) / pg * pg;
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return nullptr;
    unsigned long mask[16] = {0};  // nodes 0..1023
    if (node < 0 || node >= 1024) {
        munmap(p, len);
        return nullptr;
    }
    mask[node / 64] = 1ul << (node % 64);
    const long MPOL_PREFERRED_ = 1;
    *bound = syscall(SYS_mbind, p, len, MPOL_PREFERRED_, mask, (unsigned long)(sizeof mask * 8), 0ul) == 0;
    if (cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
        cudaGetLastError();
        munmap(p, len);
        return nullptr;
    }
    *map_bytes = len;
    return static_cast<uint8_t *>(p);
}

// Pinned, device-mapped host memory on `node` (>= 0) or with the default
// placement (cudaHostAlloc).  *map_bytes > 0 marks the mmap'ed kind;
// *bound_node = the node mbind took, else -1.
uint8_t *pinned_alloc(uint64_t bytes, int node, uint64_t *map_bytes, int *bound_node) {
    *map_bytes = 0;
    *bound_node = -1;
    uint8_t *p = nullptr;
    if (node >= 0) {
        bool bound = false;
        p = numa_pinned_alloc(bytes ? bytes : 1, node, map_bytes, &bound);
        if (p && bound) *bound_node = node;
    }
    if (!p) {
        *map_bytes = 0;
        if (cudaHostAlloc(reinterpret_cast<void **>(&p), bytes ? bytes : 1,
                          cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    }
    return p;
}

void pinned_free(uint8_t *p, uint64_t map_bytes) {
    if (!p) return;
    if (map_bytes) {
        cudaHostUnregister(p);
        munmap(p, map_bytes);
    } else {
        cudaFreeHost(p);
    }
}

}  // namespace

uint64_t crum_launch_count(const crum_ctx *c) { return c ? c->launches : 0; }

int crum_config_init(crum_config *cfg) {
    if (!cfg) return CRUM_E_INVAL;
    cfg->chunk_bytes = 0;
    cfg->pinned_pool_bytes = 0;
    cfg->numa_node = CRUM_NUMA_AUTO;
    cfg->flags = 0;
    return CRUM_OK;
}

int crum_create(int device, const crum_config *cfg, crum_ctx **out) {
    if (!out) return CRUM_E_INVAL;
    *out = nullptr;
    const uint32_t kCfgFlags = CRUM_CFG_TIMING | CRUM_CFG_NO_GRAPH | CRUM_CFG_FUSED | CRUM_CFG_TRACE | CRUM_CFG_NO_MAPPED;
    if (cfg && ((cfg->flags & ~kCfgFlags) || (cfg->chunk_bytes % 4096) || (cfg->pinned_pool_bytes % 4096) ||
                cfg->numa_node < CRUM_NUMA_DEFAULT || cfg->numa_node >= 1024)) {
        set_detail("bad crum_config");
        return CRUM_E_INVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        set_detail("no CUDA device %d", device);
        return CRUM_E_DEVICE;
    }
    crum_ctx *c = new (std::nothrow) crum_ctx();
    if (!c) return CRUM_E_NOMEM;
    c->device = device;
    if (cfg && cfg->chunk_bytes) c->chunk = cfg->chunk_bytes;
    c->timing_cfg = cfg && (cfg->flags & CRUM_CFG_TIMING);
    c->graphs_on = !(cfg && (cfg->flags & CRUM_CFG_NO_GRAPH));
    c->fused_cfg = cfg && (cfg->flags & CRUM_CFG_FUSED);
    c->mapped_cfg = !(cfg && (cfg->flags & CRUM_CFG_NO_MAPPED));
    c->trace = cfg && (cfg->flags & CRUM_CFG_TRACE);
    auto fail = [&](int st) {
        crum_destroy(c);
        return st;
    };
    if (cudaSetDevice(device) != cudaSuccess) return fail(CRUM_E_CUDA);
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    // pinned images go to the host node of the GPU's PCIe root (multi-socket
    // boxes: the D2H/H2D traffic then never crosses the socket link);
    // crum_config.numa_node overrides (CRUM_NUMA_DEFAULT: default placement)
    const int want_node = cfg ? cfg->numa_node : CRUM_NUMA_AUTO;
    c->numa_node = want_node == CRUM_NUMA_AUTO ? device_numa_node(device) : want_node == CRUM_NUMA_DEFAULT ? -1 : want_node;
    if (cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess) return fail(CRUM_E_CUDA);
    {
        // gathers of the host path get the highest priority so their blocks are
        // dispatched ahead of the (long, persistent) detect of later ranges
        int lo_prio = 0, hi_prio = 0;
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
        if (cudaStreamCreateWithPriority(&c->gstream, cudaStreamNonBlocking, hi_prio) != cudaSuccess)
            return fail(CRUM_E_CUDA);
    }
    for (int i = 0; i < 3 * kMaxRanges; ++i)
        if (cudaEventCreate(&c->ev_trace[i]) != cudaSuccess) return fail(CRUM_E_CUDA);
    for (int i = 0; i < kRing; ++i) {
        if (cudaEventCreateWithFlags(&c->ev_gather[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming) != cudaSuccess)
            return fail(CRUM_E_CUDA);
    }
    for (int i = 0; i < kMaxRanges; ++i)
        if (cudaEventCreateWithFlags(&c->ev_range[i], cudaEventDisableTiming) != cudaSuccess) return fail(CRUM_E_CUDA);
    for (int i = 0; i < 6; ++i)
        if (cudaEventCreate(&c->ev_t[i]) != cudaSuccess) return fail(CRUM_E_CUDA);
    if (cudaEventCreateWithFlags(&c->ev_meta, cudaEventDisableTiming) != cudaSuccess) return fail(CRUM_E_CUDA);
    if (cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess) return fail(CRUM_E_CUDA);
    if (cudaStreamCreateWithFlags(&c->gcap, cudaStreamNonBlocking) != cudaSuccess) return fail(CRUM_E_CUDA);
    {
        // keep freed stream-ordered allocations in the device's default pool
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            // first use of the pool costs milliseconds: pay it here, not in a fault
            void *w = nullptr;
            if (cudaMallocAsync(&w, 8ull << 20, c->gcap) == cudaSuccess) cudaFreeAsync(w, c->gcap);
            cudaStreamSynchronize(c->gcap);
        }
        cudaGetLastError();
    }
    if (cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return fail(CRUM_E_CUDA);
    if (cudaMalloc(&c->d_st, sizeof(DevStats)) != cudaSuccess) return fail(CRUM_E_NOMEM);
    if (cudaMalloc(&c->d_rb, sizeof(RangeTotals) * (kMaxRanges + 1)) != cudaSuccess) return fail(CRUM_E_NOMEM);
    if (cudaMalloc(&c->d_done, 16) != cudaSuccess) return fail(CRUM_E_NOMEM);
    c->fused_bps = fused_blocks_per_sm();
    c->small_bps = small_blocks_per_sm();
    // bitmap | 64 B of barrier words (+ the CRUM_SMALL_STAMPS profiling stamps)
    if (cudaMalloc(&c->d_small, 4 * kSmallPages / 32 + 64 + 8 * 8 * 2048) != cudaSuccess) return fail(CRUM_E_NOMEM);
    cudaMemset(c->d_small, 0, 4 * kSmallPages / 32 + 64 + 8 * 8 * 2048);
    if (cudaHostAlloc(&c->h_st, sizeof(DevStats), cudaHostAllocMapped) != cudaSuccess) return fail(CRUM_E_NOMEM);
    if (cudaHostAlloc(&c->h_rb, sizeof(RangeTotals) * (kMaxRanges + 1), cudaHostAllocMapped) != cudaSuccess)
        return fail(CRUM_E_NOMEM);
    if (cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->dh_st), c->h_st, 0) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->dh_rb), c->h_rb, 0) != cudaSuccess)
        return fail(CRUM_E_CUDA);
    cudaMemset(c->d_st, 0, sizeof(DevStats));
    cudaMemset(c->d_rb, 0, sizeof(RangeTotals) * (kMaxRanges + 1));
    cudaMemset(c->d_done, 0, 16);
    std::vector<uint64_t> none;
    int st = rebuild(c, {}, none);
    if (st) return fail(st);
    if (cfg && cfg->pinned_pool_bytes) {
        PinnedPool *pool = new (std::nothrow) PinnedPool();
        if (!pool) return fail(CRUM_E_NOMEM);
        pool->base = pinned_alloc(cfg->pinned_pool_bytes, c->numa_node, &pool->map_bytes, &pool->numa_node);
        if (!pool->base) {
            delete pool;
            set_detail("pinned pool of %llu bytes could not be allocated",
                       (unsigned long long)cfg->pinned_pool_bytes);
            return fail(CRUM_E_NOMEM);
        }
        pool->bytes = cfg->pinned_pool_bytes;
        pool->free_ext.emplace(0, pool->bytes);
        c->pool = pool;
    }
    *out = c;
    return CRUM_OK;
}

int crum_pinned_pool_info(crum_ctx *c, uint64_t *bytes, uint64_t *in_use, uint64_t *largest, uint32_t *images) {
    if (!c) return CRUM_E_INVAL;
    PinnedPool *p = c->pool;
    if (bytes) *bytes = p ? p->bytes : 0;
    if (largest) *largest = p ? p->largest_free() : 0;
    if (p) {
        std::lock_guard<std::mutex> g(p->mu);
        if (in_use) *in_use = p->in_use;
        if (images) *images = p->images;
    } else {
        if (in_use) *in_use = 0;
        if (images) *images = 0;
    }
    return CRUM_OK;
}

int crum_destroy(crum_ctx *c) {
    if (!c) return CRUM_E_INVAL;
    NOT_IN_SESSION(c);
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto &h : c->regs) cudaFree(h.shadow);
    dev_free(c->d_regs);
    dev_free(c->d_cmp_idx);
    dev_free(c->d_cmp_seg);
    dev_free(c->d_hash_idx);
    dev_free(c->d_hash_grp);
    dev_free(c->d_big_idx);
    dev_free(c->d_big_pg);
    dev_free(c->d_force);
    dev_free(c->d_flags);
    dev_free(c->d_newhash);
    dev_free(c->d_gids);
    dev_free(c->d_sunit);
    dev_free(c->d_u2s);
    dev_free(c->d_lids);
    dev_free(c->d_lhash);
    dev_free(c->d_blk_units);
    dev_free(c->d_dbg);
    dev_free(c->d_tile_base);
    dev_free(c->d_status);
    dev_free(c->d_small);
    dev_free(c->d_reg_nd);
    dev_free(c->d_rs);
    dev_free(c->d_tregs);
    dev_free(c->d_rb);
    dev_free(c->d_done);
    dev_free(c->d_zsz);
    dev_free(c->d_zloc);
    dev_free(c->d_rtmp);
    dev_free(c->d_renc);
    dev_free(c->d_zblk);
    dev_free(c->d_zrun);
    if (c->h_zrun) cudaFreeHost(c->h_zrun);
    dev_free(c->d_zbase);
    dev_free(c->d_zstage);
    dev_free(c->d_zraw);
    dev_free(c->d_st);
    dev_free(c->d_meta);
    for (int i = 0; i < kRing; ++i) dev_free(c->d_ring[i]);
    if (c->h_st) cudaFreeHost(c->h_st);
    if (c->h_rb) cudaFreeHost(c->h_rb);
    if (c->pool) {
        pinned_free(c->pool->base, c->pool->map_bytes);
        delete c->pool;
    }
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->gstream) cudaStreamDestroy(c->gstream);
    if (c->aux) cudaStreamDestroy(c->aux);
    for (auto &g : c->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (c->gcap) cudaStreamDestroy(c->gcap);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (int i = 0; i < kRing; ++i) {
        if (c->ev_gather[i]) cudaEventDestroy(c->ev_gather[i]);
        if (c->ev_copy[i]) cudaEventDestroy(c->ev_copy[i]);
    }
    for (int i = 0; i < kMaxRanges; ++i)
        if (c->ev_range[i]) cudaEventDestroy(c->ev_range[i]);
    for (int i = 0; i < 6; ++i)
        if (c->ev_t[i]) cudaEventDestroy(c->ev_t[i]);
    if (c->ev_meta) cudaEventDestroy(c->ev_meta);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    for (int i = 0; i < 3 * kMaxRanges; ++i)
        if (c->ev_trace[i]) cudaEventDestroy(c->ev_trace[i]);
    cudaGetLastError();
    delete c;
    return CRUM_OK;
}

namespace {

// Checks of one region descriptor that need no other region (crum.h
// preconditions); on success fills h (without shadow, id or page base).
int validate_region(crum_ctx *c, const crum_region_desc &d, HostRegion &h) {
    if (!d.ptr || d.bytes == 0) {
        set_detail("null pointer or zero bytes");
        return CRUM_E_INVAL;
    }
    if (d.page_size < 4096 || d.page_size > (2u << 20) || (d.page_size & (d.page_size - 1))) {
        set_detail("page_size %llu not a power of two in [4096, 2 MiB]", (unsigned long long)d.page_size);
        return CRUM_E_INVAL;
    }
    if (reinterpret_cast<uintptr_t>(d.ptr) % 16) {
        set_detail("ptr not 16-byte aligned");
        return CRUM_E_INVAL;
    }
    if (d.mode != CRUM_MODE_COMPARE && d.mode != CRUM_MODE_HASH_XXH3 && d.mode != CRUM_MODE_TRACKED) {
        set_detail("bad mode %u", d.mode);
        return CRUM_E_INVAL;
    }
    const uint64_t n = d.bytes / d.page_size + (d.bytes % d.page_size != 0);
    if (n > 0xffffffffull) {
        set_detail("too many pages");
        return CRUM_E_INVAL;
    }
    const uintptr_t lo = reinterpret_cast<uintptr_t>(d.ptr), hi = lo + d.bytes;
    if (hi < lo) return CRUM_E_INVAL;
    for (uintptr_t a : {lo, hi - 1}) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, reinterpret_cast<void *>(a)) != cudaSuccess) {
            cudaGetLastError();
            set_detail("pointer %p is not a CUDA pointer", reinterpret_cast<void *>(a));
            return CRUM_E_DEVICE;
        }
        // device memory of this device, managed memory, or pinned host memory
        // mapped at the same address (UVA): host-resident pages the kernels
        // read over the host link (oversubscribed footprints, config 5)
        const bool ok = (at.type == cudaMemoryTypeManaged) ||
                        (at.type == cudaMemoryTypeDevice && at.device == c->device) ||
                        (at.type == cudaMemoryTypeHost && at.devicePointer == reinterpret_cast<void *>(a));
        if (!ok) {
            set_detail("pointer %p is not device/managed memory of device %d", reinterpret_cast<void *>(a),
                       c->device);
            return CRUM_E_DEVICE;
        }
    }
    h = HostRegion{};
    h.mode = d.mode;
    h.ptr = static_cast<uint8_t *>(d.ptr);
    h.bytes = d.bytes;
    h.page_size = d.page_size;
    h.n_pages = n;
    h.log2p = (uint32_t)__builtin_ctzll(d.page_size);
    return CRUM_OK;
}

}  // namespace

int crum_register_regions(crum_ctx *ctx, uint32_t n, const crum_region_desc *descs, uint32_t *ids_out,
                          uint32_t *failed_index_out) {
    ENTER(ctx);
    NOT_IN_SESSION(c);
    if (failed_index_out) *failed_index_out = UINT32_MAX;
    if (n == 0) return CRUM_OK;
    if (!descs || !ids_out) {
        set_detail("null descriptor or id array");
        return CRUM_E_INVAL;
    }
    std::vector<HostRegion> add(n);
    uint64_t pages = 0;
    for (uint32_t k = 0; k < n; ++k) {
        int st = validate_region(c, descs[k], add[k]);
        if (st) {
            if (failed_index_out) *failed_index_out = k;
            return st;
        }
        pages += add[k].n_pages;
    }
    if (c->N + pages > kMaxTotalPages) {
        set_detail("too many pages");
        return CRUM_E_INVAL;
    }
    // overlap: among the batch and against the live regions (sorted sweep)
    {
        std::vector<std::pair<uintptr_t, int64_t>> iv;  // (start, batch index or -1 - live index)
        iv.reserve(n + c->regs.size());
        for (uint32_t k = 0; k < n; ++k) iv.push_back({reinterpret_cast<uintptr_t>(add[k].ptr), (int64_t)k});
        for (size_t r = 0; r < c->regs.size(); ++r)
            iv.push_back({reinterpret_cast<uintptr_t>(c->regs[r].ptr), -1 - (int64_t)r});
        std::sort(iv.begin(), iv.end());
        auto end_of = [&](int64_t t) {
            const HostRegion &h = t >= 0 ? add[t] : c->regs[-1 - t];
            return reinterpret_cast<uintptr_t>(h.ptr) + h.bytes;
        };
        for (size_t i = 1; i < iv.size(); ++i) {
            if (iv[i].first < end_of(iv[i - 1].second)) {
                const int64_t a = iv[i - 1].second, b = iv[i].second;
                const int64_t k = b >= 0 ? b : a;  // a batch entry is involved (live regions never overlap)
                if (failed_index_out) *failed_index_out = (uint32_t)k;
                if (a < 0 || b < 0) set_detail("descriptor %lld overlaps region %u", (long long)k,
                                               c->regs[-1 - (a < 0 ? a : b)].id);
                else set_detail("descriptors %lld and %lld overlap", (long long)a, (long long)b);
                return CRUM_E_OVERLAP;
            }
        }
    }
    CK(cudaDeviceSynchronize());
    // shadows: compare -> byte mirror, hash -> u64 table, tracked -> none
    int st = CRUM_OK;
    auto free_shadows = [&]() {
        for (HostRegion &h : add)
            if (h.shadow) {
                cudaFree(h.shadow);
                h.shadow = nullptr;
            }
    };
    for (uint32_t k = 0; k < n && !st; ++k) {
        HostRegion &h = add[k];
        const uint64_t shadow_bytes =
            h.mode == kModeCompare ? round_up(h.bytes, 256) : h.mode == kModeHash ? 8 * h.n_pages : 0;
        h.shadow = nullptr;
        if (shadow_bytes) {
            if ((st = dev_alloc(c, &h.shadow, shadow_bytes))) break;
            if (cudaMemset(h.shadow, 0, shadow_bytes) != cudaSuccess) {
                cudaGetLastError();
                st = CRUM_E_NOMEM;
            }
        }
    }
    if (st) {
        free_shadows();
        return st;
    }
    std::vector<uint64_t> old_base;
    for (const HostRegion &o : c->regs) old_base.push_back(o.page_base);
    std::vector<HostRegion> regs = c->regs;
    for (uint32_t k = 0; k < n; ++k) {
        add[k].id = c->next_id + k;
        regs.push_back(add[k]);
        old_base.push_back(UINT64_MAX);
    }
    st = rebuild(c, std::move(regs), old_base);
    if (st) {  // nothing changed (rebuild is transactional)
        free_shadows();
        return st;
    }
    for (uint32_t k = 0; k < n; ++k) ids_out[k] = c->next_id + k;
    c->next_id += n;
    return CRUM_OK;
}

int crum_register_region(crum_ctx *ctx, void *ptr, uint64_t bytes, uint64_t page_size, uint32_t mode,
                         uint32_t *region_id_out) {
    if (!region_id_out) {
        set_detail("null region id pointer");
        return CRUM_E_INVAL;
    }
    const crum_region_desc d{ptr, bytes, page_size, mode, 0};
    return crum_register_regions(ctx, 1, &d, region_id_out, nullptr);
}

int crum_unregister_region(crum_ctx *ctx, uint32_t id) {
    ENTER(ctx);
    NOT_IN_SESSION(c);
    uint32_t idx;
    if (!find_region(c, id, &idx)) {
        set_detail("no region %u", id);
        return CRUM_E_NOREGION;
    }
    CK(cudaDeviceSynchronize());
    std::vector<uint64_t> old_base;
    for (uint32_t r = 0; r < c->regs.size(); ++r)
        if (r != idx) old_base.push_back(c->regs[r].page_base);
    const HostRegion gone = c->regs[idx];
    std::vector<HostRegion> regs = c->regs;
    regs.erase(regs.begin() + idx);
    int st = rebuild(c, std::move(regs), old_base);
    if (st) return st;  // the region stays registered (rebuild is transactional)
    cudaFree(gone.shadow);
    return CRUM_OK;
}

int crum_mark_dirty(crum_ctx *ctx, uint32_t id, uint64_t off, uint64_t len) {
    ENTER(ctx);
    HostRegion *h = find_region(c, id);
    if (!h) {
        set_detail("no region %u", id);
        return CRUM_E_NOREGION;
    }
    if (off > h->bytes || len > h->bytes - off) {
        set_detail("range [%llu, +%llu) outside region of %llu bytes", (unsigned long long)off,
                   (unsigned long long)len, (unsigned long long)h->bytes);
        return CRUM_E_RANGE;
    }
    if (!len) return CRUM_OK;
    const uint64_t i0 = off / h->page_size, i1 = (off + len - 1) / h->page_size;
    // device-synchronous: ordered after every earlier call on any stream and
    // visible to every later one
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(c->d_force + h->page_base + i0, 1, i1 - i0 + 1));
    CK(cudaDeviceSynchronize());
    return CRUM_OK;
}

int crum_mark_dirty_pages(crum_ctx *ctx, uint32_t id, const uint32_t *dev_pages, uint64_t n, void *stream) {
    ENTER(ctx);
    HostRegion *h = find_region(c, id);
    if (!h) {
        set_detail("no region %u", id);
        return CRUM_E_NOREGION;
    }
    if (!n) return CRUM_OK;
    if (!dev_pages) {
        set_detail("null page list");
        return CRUM_E_INVAL;
    }
    launch_mark_pages(launch_of(c, static_cast<cudaStream_t>(stream)), c->d_force + h->page_base, h->n_pages,
                      dev_pages, n);
    CK_LAUNCH();
    return CRUM_OK;
}

int crum_region_tracker(crum_ctx *ctx, uint32_t id, crum_tracker *out) {
    ENTER(ctx);
    HostRegion *h = find_region(c, id);
    if (!h) {
        set_detail("no region %u", id);
        return CRUM_E_NOREGION;
    }
    if (!out) return CRUM_E_INVAL;
    out->force = c->d_force + h->page_base;
    out->bytes = h->bytes;
    out->log2_page = h->log2p;
    out->reserved = 0;
    return CRUM_OK;
}

int crum_image_required_bytes(crum_ctx *ctx, uint64_t max_dirty, uint64_t *out) {
    ENTER(ctx);
    if (!out) return CRUM_E_INVAL;
    const uint64_t K = std::min(max_dirty, c->N);
    uint64_t payload = 0, maxp = 0;
    for (const HostRegion &h : c->regs) {
        payload += h.n_pages * h.page_size;
        maxp = std::max(maxp, h.page_size);
    }
    if (K < c->N && K * maxp < payload) payload = K * maxp;
    // + the unit-size table of a compressed image (an encoded unit is never
    // longer than the unit)
    *out = payload_offset_for(c->regs.size()) + payload + tail_bytes_for(K, c->any_hash) +
           round_up(2 * (payload >> kSegLog2), 8);
    return CRUM_OK;
}


int crum_device_numa_node(int device, int *node_out) {
    if (!node_out) return CRUM_E_INVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        set_detail("no CUDA device %d", device);
        return CRUM_E_DEVICE;
    }
    *node_out = device_numa_node(device);
    return CRUM_OK;
}

int crum_image_numa_node(const crum_image *img, int *node_out) {
    if (!img || !node_out) return CRUM_E_INVAL;
    *node_out = img->numa_node;
    return CRUM_OK;
}

int crum_image_create(crum_ctx *ctx, uint64_t cap, crum_image **out) {
    ENTER(ctx);
    if (!out) return CRUM_E_INVAL;
    crum_image *im = new (std::nothrow) crum_image{nullptr, cap, 0, c->device};
    if (!im) return CRUM_E_NOMEM;
    if (c->pool && (im->host = c->pool->carve(cap))) {
        im->pool = c->pool;
        im->numa_node = c->pool->numa_node;
    } else {
        im->host = pinned_alloc(cap, c->numa_node, &im->map_bytes, &im->numa_node);
    }
    if (!im->host) {
        delete im;
        set_detail("pinned allocation of %llu bytes failed", (unsigned long long)cap);
        return CRUM_E_NOMEM;
    }
    *out = im;
    return CRUM_OK;
}

int crum_image_import(crum_ctx *ctx, const void *bytes, uint64_t len, crum_image **out) {
    if (!bytes && len) return CRUM_E_INVAL;
    int st = crum_image_create(ctx, len, out);
    if (st) return st;
    if (len) memcpy((*out)->host, bytes, len);
    (*out)->len = len;
    return CRUM_OK;
}

int crum_image_data(const crum_image *img, void **data, uint64_t *len, uint64_t *cap) {
    if (!img || !data || !len) return CRUM_E_INVAL;
    *data = img->host;
    *len = img->len;
    if (cap) *cap = img->cap;
    return CRUM_OK;
}

int crum_image_destroy(crum_image *img) {
    if (!img) return CRUM_E_INVAL;
    if (img->sessions) {
        set_detail("a lazy restore session reads this image");
        return CRUM_E_BUSY;
    }
    if (img->writer.joinable()) img->writer.join();
    cudaSetDevice(img->device);
    if (img->pool) img->pool->release(img->host, img->cap);
    else pinned_free(img->host, img->map_bytes);
    delete img;
    return CRUM_OK;
}

namespace {
// Write all of [p, p+n) to fd (short writes and EINTR handled).
bool write_all(int fd, const uint8_t *p, uint64_t n) {
    while (n) {
        const ssize_t w = ::write(fd, p, std::min<uint64_t>(n, 1ull << 30));
        if (w < 0) {
            if (errno == EINTR) continue;
            return false;
        }
        p += w;
        n -= (uint64_t)w;
    }
    return true;
}
}  // namespace

int crum_image_persist(crum_image *img, const char *path, uint32_t flags) {
    if (!img || !path || (flags & ~(uint32_t)(CRUM_PERSIST_FSYNC | CRUM_PERSIST_DIRECT))) {
        set_detail("null image/path or bad flags");
        return CRUM_E_INVAL;
    }
    if (img->busy.load()) {
        set_detail("image is being persisted");
        return CRUM_E_BUSY;
    }
    if (img->writer.joinable()) img->writer.join();
    img->busy.store(1);
    img->result = CRUM_OK;
    img->error.clear();
    const std::string dst(path);
    img->writer = std::thread([img, dst, flags]() {
        const bool direct = flags & CRUM_PERSIST_DIRECT;
        const int fd = ::open(dst.c_str(), O_WRONLY | O_CREAT | O_TRUNC | (direct ? O_DIRECT : 0), 0644);
        bool ok = fd >= 0;
        if (ok && !direct) ok = write_all(fd, img->host, img->len);
        if (ok && direct) {
            // whole 4 KiB blocks straight from the (page-aligned) pinned image;
            // the last partial block through an aligned bounce block
            constexpr uint64_t kBlk = 4096;
            const uint64_t whole = img->len / kBlk * kBlk, rest = img->len - whole;
            ok = write_all(fd, img->host, whole);
            if (ok && rest) {
                void *b = nullptr;
                ok = posix_memalign(&b, kBlk, kBlk) == 0;
                if (ok) {
                    memset(b, 0, kBlk);
                    memcpy(b, img->host + whole, rest);
                    ok = write_all(fd, static_cast<const uint8_t *>(b), kBlk);
                    free(b);
                }
            }
            if (ok) ok = ::ftruncate(fd, (off_t)img->len) == 0;
        }
        if (ok && (flags & CRUM_PERSIST_FSYNC)) ok = ::fsync(fd) == 0;
        if (fd >= 0 && ::close(fd) != 0) ok = false;
        if (!ok) {
            img->result = CRUM_E_IO;
            img->error = "persist " + dst + ": " + strerror(errno);
        }
        img->busy.store(0);
    });
    return CRUM_OK;
}

int crum_image_persist_wait(crum_image *img) {
    if (!img) return CRUM_E_INVAL;
    if (img->writer.joinable()) img->writer.join();
    if (img->result != CRUM_OK) set_detail("%s", img->error.c_str());
    return img->result;
}

int crum_image_persist_busy(const crum_image *img, int *busy_out) {
    if (!img || !busy_out) return CRUM_E_INVAL;
    *busy_out = img->busy.load();
    return CRUM_OK;
}

int crum_image_load(crum_ctx *ctx, const char *path, crum_image **out) {
    if (!path || !out) return CRUM_E_INVAL;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) {
        set_detail("open %s: %s", path, strerror(errno));
        return CRUM_E_IO;
    }
    struct stat sb;
    if (::fstat(fd, &sb) != 0) {
        ::close(fd);
        set_detail("stat %s: %s", path, strerror(errno));
        return CRUM_E_IO;
    }
    const uint64_t len = (uint64_t)sb.st_size;
    int st = crum_image_create(ctx, len, out);
    if (st) {
        ::close(fd);
        return st;
    }
    uint8_t *p = (*out)->host;
    uint64_t n = len;
    while (n) {
        const ssize_t r = ::read(fd, p, std::min<uint64_t>(n, 1ull << 30));
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) {
            ::close(fd);
            crum_image_destroy(*out);
            *out = nullptr;
            set_detail("read %s: %s", path, r < 0 ? strerror(errno) : "short file");
            return CRUM_E_IO;
        }
        p += r;
        n -= (uint64_t)r;
    }
    ::close(fd);
    (*out)->len = len;
    return CRUM_OK;
}

// ---------------------------------------------------------------------------
// A7: sync shadow = detect + compact + commit (no image)
// ---------------------------------------------------------------------------
namespace {
// A1-A3 into a device image (stream-ordered): detect, compact (+ table,
// header fields), gather (+ commit), and on the side stream the metadata CRC
// (+ tail, header).
// Timing / completion events are recorded as external event nodes so they
// also fire when the sequence runs as a captured graph.
// The single-pass kernel (detect + compaction + gather + commit, then the
// metadata CRC) runs when the context asked for it (CRUM_CFG_FUSED) and, by
// default, for footprints up to kFusedSmallBytes: there the multi-kernel
// sequence is latency-bound (C1: detect -> compaction -> CRC, each a few
// dependent round trips) and one launch removes two of them.  Eligible: all
// regions COMPARE with pages <= 64 KiB, an incremental gather, and an image
// that holds the worst case (no capacity failure can occur mid-kernel).
// Above kFusedSmallBytes the single pass also runs when the previous
// checkpoint listed at least kFusedDirtyFrac of the pages: it reads each dirty
// page once (2F + 2KP) where the multi-kernel path re-reads it (2F + 3KP) --
// measured on C2 compare, device image: d = 1: 1760 vs 1201 GB/s; d = 0.1:
// 2473 vs 2667 GB/s (profiles/r02/sweep/).  The previous call's K is read
// from the mapped copy of its stats (possibly one call older: a heuristic only;
// both paths produce the same image).
constexpr double kFusedDirtyFrac = 0.25;

// The single pass L2-prefetches each tile's next segment unless the previous
// checkpoint listed >= kFusedDirtyFrac of a large footprint (C2,
// profiles/r02/fused_prefetch_ab/: kernel d = 1 % 0.87 vs 0.83 of peak,
// 10 % 0.93 vs 0.87, 100 % 1.10 vs 1.12).  A heuristic on the mapped stats.
bool fused_prefetch(const crum_ctx *c) {
    const uint64_t prev_k = *reinterpret_cast<volatile const uint64_t *>(&c->h_st->K);
    return !(c->N && c->F > kFusedSmallBytes && (double)prev_k >= kFusedDirtyFrac * (double)c->N);
}

bool use_fused(const crum_ctx *c, bool full, uint64_t capacity, uint64_t worst) {
    if (!c->fused_ok || full || capacity < worst) return false;
    if (c->fused_cfg || c->F <= kFusedSmallBytes) return true;
    const uint64_t prev_k = *reinterpret_cast<volatile const uint64_t *>(&c->h_st->K);
    return c->N && prev_k <= c->N && (double)prev_k >= kFusedDirtyFrac * (double)c->N;
}

// The one-launch small path (k_small_ckpt): preferred over the single-pass
// kernel where it applies (one page size, COMPARE / TRACKED, N <= kSmallPages).
bool use_small(const crum_ctx *c, bool full, uint64_t capacity, uint64_t worst) {
    return c->small_ok && !full && capacity >= worst;
}

int enqueue_small(crum_ctx *c, cudaStream_t s, uint8_t *img, uint64_t capacity, bool timing, bool capturing = false) {
    const unsigned evf = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    SmallArgs sa{};
    sa.timing = timing;  // the kernel times itself: no events around it
    sa.regs = c->d_regs;
    sa.R = (uint32_t)c->regs.size();
    sa.log2p = c->small_log2p;
    sa.N = c->N;
    sa.bitmap = c->d_small;
    sa.bar = c->d_small + kSmallPages / 32;
    sa.force = c->d_force;
    sa.img = img;
    sa.poff = payload_offset_for(c->regs.size());
    sa.capacity = capacity;
    sa.st = c->d_st;
    sa.st_host = c->dh_st;
    sa.x2n = crc_tables().x2n;
    const uint64_t warps = (c->N << (c->small_log2p - kSegLog2)) << kSmallItemsLog2;  // a detect item each
    uint64_t blocks = (warps + 7) / 8 + 1;  // + CTA 0 (metadata; it detects nothing)
    const uint64_t cap = (uint64_t)c->sms * c->small_bps;  // co-resident (cooperative launch)
    if (blocks > cap) blocks = cap;
    if (blocks < 2) blocks = 2;  // CTA 0 writes the metadata beside the gathers of the others
    if (blocks > cap) blocks = cap;
    Launch L = launch_of(c, s);
    launch_small_ckpt(L, sa, (int)blocks);
    CK_LAUNCH();
    CK(cudaEventRecordWithFlags(c->ev_done, s, evf));
    return CRUM_OK;
}

// Stream-ordered and graph-capturable: the scratch, per-region counts and
// look-back status words are cleared before every launch (status words carry
// a constant tag).
// meta != nullptr: img is a pinned image's mapped address; the region table
// goes to meta (device) and k_crc_meta copies table + padding, writes the tail
// and header into img (never reading the image back across the host link).
int enqueue_fused(crum_ctx *c, cudaStream_t s, uint8_t *img, uint64_t capacity, bool timing, bool capturing = false,
                  uint8_t *meta = nullptr) {
    const unsigned evf = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[0], s, evf));
    const uint64_t R = c->regs.size();
    CK(cudaMemsetAsync(c->d_status, 0, fused_scratch_bytes(R, c->n_tiles), s));
    uint8_t *scr = reinterpret_cast<uint8_t *>(c->d_status);
    FusedArgs fa{};
    fa.regs = c->d_regs;
    fa.R = (uint32_t)R;
    fa.tag = 1;
    fa.tile_log2_min = c->fused_tile_min;
    fa.inline_meta = !meta && c->F <= kFusedSmallBytes && 48 * R + 4 * c->N + 8 <= kFusedInlineMeta;
    fa.prefetch = fused_prefetch(c) ? 1 : 0;
    fa.meta = meta;
    fa.x2n = crc_tables().x2n;
    fa.tile_base = c->d_tile_base;
    fa.n_tiles = c->n_tiles;
    fa.fs = reinterpret_cast<FusedScratch *>(scr);
    fa.reg_nd = reinterpret_cast<uint32_t *>(scr + kFsHead);
    fa.status = reinterpret_cast<uint64_t *>(scr + kFsHead + fused_counts_bytes(R));
    fa.force = c->d_force;
    fa.img = img;
    fa.poff = payload_offset_for(c->regs.size());
    fa.gids = c->d_gids;
    fa.sunit = c->d_sunit;
    fa.lids = c->d_lids;
    fa.rs = c->d_rs;
    fa.st = c->d_st;
    fa.st_host = c->dh_st;
    fa.capacity = capacity;
    Launch L = launch_of(c, s);
    launch_fused_compare(L, fa, c->sms * c->fused_bps);
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[1], s, evf));
    if (!fa.inline_meta) {  // stats -> mapped (use_fused)
        CrcArgs cra = crc_args(c, meta ? meta : img, nullptr);
        cra.out = meta ? img : nullptr;
        launch_crc_meta(L, cra, crc_max_len(c));
    }
    CK_LAUNCH();
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[4], s, evf));
    CK(cudaEventRecordWithFlags(c->ev_done, s, evf));
    return CRUM_OK;
}

int enqueue_gather_dev(crum_ctx *c, cudaStream_t s, uint8_t *img, uint64_t capacity, bool full, bool timing,
                       bool capturing = false) {
    const unsigned evf = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[0], s, evf));
    CK(cudaMemsetAsync(c->d_rb, 0, sizeof(RangeTotals), s));
    enqueue_detect(c, s, c->all, full);
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[1], s, evf));
    // device path: no mapped-host mirrors of the totals (only the host pipeline reads them)
    CompactArgs ca = compact_args(c, c->all, 0, true, true, full, capacity, img);
    ca.rb_host = nullptr;
    enqueue_compact(c, s, ca);
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[2], s, evf));
    // metadata CRC (+ tail, header) on a side stream beside the payload gather
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
    CrcArgs cra = crc_args(c, img, nullptr);  // st_host: the stats reach mapped memory (use_fused)
    launch_crc_meta(launch_of(c, c->aux), cra, crc_max_len(c));
    CK(cudaEventRecord(c->ev_join, c->aux));
    Launch L = launch_of(c, s);
    launch_gather(L, gather_args(c, 0, img, 0, true, 0, UINT64_MAX), c->max_units);
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[3], s, evf));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    CK_LAUNCH();
    if (timing) CK(cudaEventRecordWithFlags(c->ev_t[4], s, evf));
    CK(cudaEventRecordWithFlags(c->ev_done, s, evf));
    return CRUM_OK;
}

// The same sequence as a CUDA graph: captured on the context's capture stream
// the first time a (image, capacity, flags) triple is seen in this registry
// generation, then replayed on `s`.  CRUM_E_BUSY: capture unavailable, the
// caller enqueues directly.
int gather_dev_graph(crum_ctx *c, cudaStream_t s, uint8_t *img, uint64_t capacity, uint32_t flags, bool timing) {
    uint64_t worst = 0;
    crum_image_required_bytes(c, UINT64_MAX, &worst);
    const bool small = use_small(c, (flags & CRUM_FULL) != 0, capacity, worst);
    const bool fused = !small && use_fused(c, (flags & CRUM_FULL) != 0, capacity, worst);
    // the key includes whether events are recorded and which sequence runs
    flags |= (timing ? 0x80000000u : 0u) | (fused ? 0x40000000u : 0u) | (small ? 0x20000000u : 0u) |
             (fused && fused_prefetch(c) ? 0x10000000u : 0u);
    crum_ctx::GraphEntry *e = nullptr, *victim = &c->graphs[0];
    for (auto &g : c->graphs) {
        if (g.exec && g.epoch == c->graph_epoch && g.img == img && g.cap == capacity && g.flags == flags) {
            e = &g;
            break;
        }
        if (!g.exec || g.used < victim->used) victim = &g;
    }
    if (!e) {
        e = victim;
        if (e->exec) {
            cudaGraphExecDestroy(e->exec);
            e->exec = nullptr;
        }
        const uint64_t l0 = c->launches;
        if (cudaStreamBeginCapture(c->gcap, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
            cudaGetLastError();
            return CRUM_E_BUSY;
        }
        const int st = small ? enqueue_small(c, c->gcap, img, capacity, timing, true)
                       : fused ? enqueue_fused(c, c->gcap, img, capacity, timing, true)
                               : enqueue_gather_dev(c, c->gcap, img, capacity, (flags & CRUM_FULL) != 0, timing, true);
        e->fused = small || fused;
        e->small = small;
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(c->gcap, &g);
        const uint64_t nk = c->launches - l0;
        c->launches = l0;
        if (st || ce != cudaSuccess || !g) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return st ? st : CRUM_E_BUSY;
        }
        const cudaError_t ei = cudaGraphInstantiate(&e->exec, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) {
            cudaGetLastError();
            e->exec = nullptr;
            return CRUM_E_BUSY;
        }
        e->nk = nk;
        e->epoch = c->graph_epoch;
        e->img = img;
        e->cap = capacity;
        e->flags = flags;
    }
    e->used = ++c->graph_clock;
    CK(cudaGraphLaunch(e->exec, s));
    c->launches += e->nk;
    c->last_kind = e->fused ? kLastDevFused : kLastDevGather;
    c->last_small = e->small;
    return CRUM_OK;
}

// Compressed gather (readings Z2-Z3).  Chunks of
// of 16-128 MiB of units (a quarter of a range) run on the gather stream: k_gather of the
// chunk's listed pages into a raw staging buffer (no commit), encode, chunk
// scan of the sizes (running total mirrored into mapped memory), pack.  A
// pinned image takes a range pipeline like the plain path's, on coarser
// ranges (c->zranges, from 64 MiB) and one range of detection ahead (detect +
// compact of range c on the caller's stream while chunks of range c - 1
// encode and copy); each chunk's packed bytes go through a ring slot and one D2H copy
// (the host reads the chunk's end offset once its pack is done, behind the
// next chunk's encode).  Measured alternatives (profiles/r02/compress/):
// short first chunks doubling up to 16 MiB (the link starts after a small
// encode, but every chunk costs a host round trip: C2 random 468 vs 479
// GB/s); packing straight into the pinned image through its mapped address
// (no copies, no per-chunk host wait: SM stores crossed the link at
// ~47 GB/s against the copy engine's ~53, C2 random 320 GB/s).
// A device image compacts everything first and packs in place.  Then the
// image fields (k_zfinal), the metadata CRC + tail + header (a pinned image's
// header + table are built in device memory and copied in by the CRC
// kernel), and -- only once the image is known to fit -- the commit of every
// listed page, range by range.
int gather_z(crum_ctx *c, cudaStream_t s, uint8_t *dev_img, crum_image *himg, uint64_t capacity, bool full,
             bool timing, crum_report *rep) {
    int st;
    if ((st = ensure_z(c, c->max_units))) return st;
    if (himg && (st = ensure_ring(c, (uint64_t)kZChunkUnits << kSegLog2))) return st;
    uint8_t *img = dev_img;  // device address of the image (a pinned image: its mapped address)
    if (himg) {
        void *dp = nullptr;
        CK(cudaHostGetDevicePointer(&dp, himg->host, 0));
        img = static_cast<uint8_t *>(dp);
    }
    const uint64_t poff = payload_offset_for(c->regs.size());
    uint8_t *head = himg ? c->d_meta : (capacity >= poff ? img : nullptr);
    const uint64_t plimit = capacity > poff ? capacity - poff : 1;  // payload bytes that fit
    // a host image streams range by range; a device image is one range
    const uint32_t nr = himg ? (uint32_t)c->zranges.size() : 1;
    auto range_of = [&](uint32_t ci) -> const Range & { return himg ? c->zranges[ci] : c->all; };
    Launch G = launch_of(c, c->gstream);
    CK(cudaEventRecord(c->ev_t[0], s));
    CK(cudaMemsetAsync(c->d_rb, 0, sizeof(RangeTotals), s));
    CK(cudaMemsetAsync(c->d_zrun, 0, 8, s));
    uint32_t enq = 0;
    auto enqueue_range = [&](uint32_t ci) -> int {
        enqueue_detect(c, s, range_of(ci), full);
        enqueue_compact(c, s, compact_args(c, range_of(ci), ci, ci == 0, ci + 1 == nr, full, UINT64_MAX, head));
        CK_LAUNCH();
        CK(cudaEventRecord(c->ev_range[ci], s));  // h_rb[ci + 1] written by the kernel (mapped)
        if (ci + 1 == nr) {
            CK(cudaEventRecord(c->ev_t[1], s));
            if (!himg) CK(cudaEventRecord(c->ev_t[2], s));  // device image: encoding starts here
        }
        return CRUM_OK;
    };
    // one range ahead of the chunk loop: a detect grid holds the SMs the
    // encoder needs (C2, profiles/r02/compress/lookahead/: two ahead random
    // 465 / half 602 / hpgmg 549 GB/s, one ahead 466 / 618 / 553, all ahead
    // 404 / 521 / 485)
    while (enq < nr && enq < 1)
        if ((st = enqueue_range(enq++))) return st;
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(c->gstream, c->ev_fork, 0));  // the zrun / rb resets
    c->h_zrun[0] = 0;
    c->h_rb[0] = RangeTotals{0, 0};
    uint64_t k = 0;  // chunk index
    bool overflow = false, copy_started = false;
    auto copy_chunk = [&](uint64_t kk) -> int {  // host image: chunk kk's packed bytes -> the image
        const int slot = (int)(kk % kRing);
        CK(cudaEventSynchronize(c->ev_gather[slot]));
        const uint64_t o0 = c->h_zrun[kk], o1 = c->h_zrun[kk + 1];
        if (poff + o1 > himg->cap) overflow = true;  // CAPACITY: stop copying, keep encoding for the size
        CK(cudaStreamWaitEvent(c->copy, c->ev_gather[slot], 0));
        if (!overflow && o1 > o0) {
            if (!copy_started) {
                CK(cudaEventRecord(c->ev_t[4], c->copy));
                copy_started = true;
            }
            CK(cudaMemcpyAsync(himg->host + poff + o0, c->d_ring[slot], o1 - o0, cudaMemcpyDeviceToHost, c->copy));
        }
        CK(cudaEventRecord(c->ev_copy[slot], c->copy));
        if (c->trace && kk < (uint64_t)kMaxRanges) CK(cudaEventRecord(c->ev_trace[3 * kk + 2], c->copy));
        return CRUM_OK;
    };
    for (uint32_t ci = 0; ci < nr; ++ci) {
        while (enq < nr && enq <= ci + 1)
            if ((st = enqueue_range(enq++))) return st;
        CK(cudaEventSynchronize(c->ev_range[ci]));
        const uint64_t U0 = c->h_rb[ci].units, U1 = c->h_rb[ci + 1].units;
        if (U1 > U0) CK(cudaStreamWaitEvent(c->gstream, c->ev_range[ci], 0));
        // chunks of a quarter of the range's units, 16-128 MiB: per-chunk costs
        // (kernel drains, the single-block scan, host wait) amortise over large
        // payloads, small ones keep a few chunks in flight (C4 HPGMG-like
        // compressed: 16 MiB chunks 730 GB/s, 32 MiB 794-798, 64 MiB 868,
        // 128 MiB 908; C2 hpgmg at a fixed 64 MiB 583 vs 601 at 16 MiB)
        const uint64_t cu = std::min<uint64_t>(kZChunkUnits, std::max<uint64_t>(kZMinChunkUnits, (U1 - U0) / 4));
        for (uint64_t u0 = U0; u0 < U1; u0 += cu, ++k) {
            const uint64_t u1 = std::min(U1, u0 + cu), n = u1 - u0;
            const int slot = (int)(k % kRing);
            GatherArgs ga = gather_args(c, ci, c->d_zraw, u0, false, u0, u1);
            ga.no_commit = 1;
            launch_gather(G, ga, n);
            launch_zenc(G, c->d_zraw, n, c->d_zstage, c->d_zsz + u0, c->d_st);
            if (c->trace && k < (uint64_t)kMaxRanges) CK(cudaEventRecord(c->ev_trace[3 * k], c->gstream));
            launch_zscan_chunk(G, c->d_zsz + u0, n, c->d_zloc + u0, c->d_zrun, c->d_zbase + k,
                               himg ? c->dh_zrun + k + 1 : nullptr);
            if (himg) {
                if (k >= (uint64_t)kRing) CK(cudaStreamWaitEvent(c->gstream, c->ev_copy[slot], 0));
                launch_zpack(G, c->d_zstage, c->d_zsz + u0, c->d_zloc + u0, n, nullptr, c->d_ring[slot], 0, c->d_st);
                CK_LAUNCH();
                CK(cudaEventRecord(c->ev_gather[slot], c->gstream));
                if (c->trace && k < (uint64_t)kMaxRanges) CK(cudaEventRecord(c->ev_trace[3 * k + 1], c->gstream));
                if (k && (st = copy_chunk(k - 1))) return st;
            } else {
                launch_zpack(G, c->d_zstage, c->d_zsz + u0, c->d_zloc + u0, n, c->d_zbase + k, img + poff, plimit,
                             c->d_st);
                CK_LAUNCH();
            }
        }
    }
    if (himg && k && (st = copy_chunk(k - 1))) return st;
    CK(cudaEventRecord(c->ev_t[3], c->gstream));
    if (himg && !copy_started) CK(cudaEventRecord(c->ev_t[4], c->copy));
    // image fields, CRC + tail + header, then the commit -- after the last range
    CK(cudaStreamWaitEvent(c->gstream, c->ev_range[nr - 1], 0));
    launch_zfinal(G, c->d_st, c->d_zrun, capacity >= poff ? img : nullptr, capacity);
    CrcArgs cra = crc_args(c, head, nullptr);
    cra.out = himg ? img : nullptr;
    if (head) launch_crc_meta(G, cra, crc_max_len(c));
    for (uint32_t ci = 0; ci < nr; ++ci) {
        const uint64_t U0 = c->h_rb[ci].units, U1 = c->h_rb[ci + 1].units;
        if (U1 > U0) launch_gather(G, gather_args(c, ci, nullptr, 0, false, U0, U1), U1 - U0);  // commit only
    }
    CK_LAUNCH();
    CK(cudaEventRecord(c->ev_join, c->gstream));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    if (himg) {
        CK(cudaEventRecord(c->ev_t[5], c->copy));
        CK(cudaStreamWaitEvent(s, c->ev_t[5], 0));
    } else {
        CK(cudaEventRecord(c->ev_t[4], s));  // device image: e4 = end of the call
    }
    CK(cudaEventRecord(c->ev_done, s));
    c->last_kind = himg ? kLastHostGather : kLastDevGather;
    c->last_timed = timing;
    c->last_path = CRUM_PATH_COMPRESSED;
    if (!himg && !rep) return CRUM_OK;  // stream-asynchronous (capacity >= worst case)
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost));
    const DevStats h = *c->h_st;
    if (himg && h.status == kStOk) himg->len = h.image_bytes;
    if (c->trace && himg) {
        fprintf(stderr, "[crum trace] compressed gather: %u ranges, %llu chunks, K=%llu, image=%llu B, "
                        "detect %.3f  first copy %.3f  packed %.3f  copied %.3f ms\n",
                nr, (unsigned long long)k, (unsigned long long)h.K, (unsigned long long)h.image_bytes,
                ev_ms(c->ev_t[0], c->ev_t[1]), ev_ms(c->ev_t[0], c->ev_t[4]), ev_ms(c->ev_t[0], c->ev_t[3]),
                ev_ms(c->ev_t[0], c->ev_t[5]));
        for (uint64_t kk = 0; kk < std::min<uint64_t>(k, kMaxRanges); ++kk)
            fprintf(stderr, "[crum trace]  chunk %2llu bytes %llu: encoded %.3f  packed %.3f  copied %.3f ms\n",
                    (unsigned long long)kk, (unsigned long long)(c->h_zrun[kk + 1] - c->h_zrun[kk]),
                    ev_ms(c->ev_t[0], c->ev_trace[3 * kk]), ev_ms(c->ev_t[0], c->ev_trace[3 * kk + 1]),
                    ev_ms(c->ev_t[0], c->ev_trace[3 * kk + 2]));
    }
    if (rep) {
        memset(rep, 0, sizeof *rep);
        fill_report(c, h, rep);
        fill_times(c, h, rep);
        rep->path |= CRUM_PATH_COMPRESSED;
    }
    if (h.status == kStCapacity) {
        set_detail("image needs %llu bytes, capacity %llu", (unsigned long long)h.image_bytes,
                   (unsigned long long)capacity);
        return CRUM_E_CAPACITY;
    }
    return CRUM_OK;
}

// A pinned gather with a small expected payload and an image that holds a
// worst-case image: no staging ring, no D2H copies, no host wait until the
// end.  The kernels store the payload and the metadata straight into the
// pinned image through its mapped address:
//  * fused (every region COMPARE with pages <= 64 KiB, previous payload
//    2-16 MiB): the single-pass kernel -- each tile's dirty pages cross the
//    host link as soon as the tile's look-back resolves, so the stores
//    overlap the detection of later tiles (C2 1 %: 0.58 -> 0.47 ms);
//  * split (otherwise, previous payload 1-16 MiB): detect + compact per
//    range of c->mranges (1/2, 1/4, 1/4 of the pages) on s, each range's
//    gather on the gather stream behind its compaction, so the stores of a
//    range overlap the detection of the next;
//  * otherwise one range: detect, compact, gather (mapped stores) -- at
//    <= 1 MiB the stores are short, and the detect kernel is faster than the
//    single pass (C2 0 %: 0.44 ms single pass, 0.37 ms one range).
// Then the metadata CRC kernel copies the table (kept in device memory),
// writes the tail and header into the image and the final stats into mapped
// memory; the host waits once.
int gather_mapped(crum_ctx *c, cudaStream_t s, crum_image *img, bool fused, bool split, crum_report *rep) {
    void *dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, img->host, 0));
    uint8_t *d = static_cast<uint8_t *>(dp);
    int st;
    if (fused) {
        if ((st = enqueue_fused(c, s, d, img->cap, true, false, c->d_meta))) return st;
        CK(cudaEventRecord(c->ev_t[3], s));  // (ev_t[0] / ev_t[1] / ev_t[4] recorded by enqueue_fused)
    } else {
        // per range: detect + compact on s; the range's gather on the gather
        // stream (its unit bounds read from the device totals), storing while
        // the next range is detected
        const std::vector<Range> one{c->all};
        const std::vector<Range> &rs = split ? c->mranges : one;
        const uint32_t nr = (uint32_t)rs.size();
        uint8_t *payload = d + payload_offset_for(c->regs.size());
        Launch L = launch_of(c, s), G = launch_of(c, c->gstream);
        CK(cudaEventRecord(c->ev_t[0], s));
        CK(cudaEventRecord(c->ev_t[4], s));  // the stores start with the first range's gather
        CK(cudaMemsetAsync(c->d_rb, 0, sizeof(RangeTotals), s));
        for (uint32_t ci = 0; ci < nr; ++ci) {
            enqueue_detect(c, s, rs[ci], false);
            CompactArgs ca = compact_args(c, rs[ci], ci, ci == 0, ci + 1 == nr, false, img->cap, c->d_meta);
            ca.rb_host = nullptr;
            enqueue_compact(c, s, ca);
            CK(cudaEventRecord(c->ev_range[ci], s));
            CK(cudaStreamWaitEvent(c->gstream, c->ev_range[ci], 0));
            // the stores are bound by the host link: at most one CTA per SM
            launch_gather(G, gather_args(c, ci, payload, 0, false, 0, UINT64_MAX),
                          std::min<uint64_t>(c->max_units, (uint64_t)c->sms * 64));
            CK_LAUNCH();
        }
        CK(cudaEventRecord(c->ev_t[1], s));
        CrcArgs cra = crc_args(c, c->d_meta, nullptr);
        cra.out = d;
        launch_crc_meta(L, cra, crc_max_len(c));
        CK_LAUNCH();
        CK(cudaEventRecord(c->ev_t[3], c->gstream));
        CK(cudaStreamWaitEvent(s, c->ev_t[3], 0));
    }
    CK(cudaEventRecord(c->ev_t[5], s));
    CK(cudaEventRecord(c->ev_done, s));
    CK(cudaStreamSynchronize(s));
    c->last_kind = kLastHostGather;
    c->last_timed = true;
    c->last_path = CRUM_PATH_MAPPED | (fused ? CRUM_PATH_FUSED : 0u);
    const DevStats h = *c->h_st;  // written by the CRC kernel's last block (mapped)
    img->len = h.image_bytes;
    ++c->gathers_since_rebuild;
    if (rep) {
        memset(rep, 0, sizeof *rep);
        fill_report(c, h, rep);
        fill_times(c, h, rep);
        rep->t_copy_ms = ev_ms(c->ev_t[0], c->ev_t[5]);  // the stores span the call
    }
    return CRUM_OK;
}

}  // namespace

int crum_sync_shadow(crum_ctx *ctx, void *stream, uint64_t *dirty_out) {
    NvtxRange nvtx_("crum_sync_shadow");
    ENTER(ctx);
    NOT_IN_SESSION(c);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool timing = c->timing_cfg;
    if (timing) CK(cudaEventRecord(c->ev_t[0], s));
    CK(cudaMemsetAsync(c->d_rb, 0, sizeof(RangeTotals), s));
    enqueue_detect(c, s, c->all, false);
    if (timing) CK(cudaEventRecord(c->ev_t[1], s));
    CompactArgs ca = compact_args(c, c->all, 0, true, true, false, UINT64_MAX, nullptr);
    ca.rb_host = nullptr;
    enqueue_compact(c, s, ca);
    if (timing) CK(cudaEventRecord(c->ev_t[2], s));
    Launch L = launch_of(c, s);
    launch_gather(L, gather_args(c, 0, nullptr, 0, false, 0, UINT64_MAX), c->max_units);
    CK_LAUNCH();
    if (timing) CK(cudaEventRecord(c->ev_t[4], s));
    CK(cudaEventRecord(c->ev_done, s));
    c->last_kind = kLastSync;
    c->last_path = 0;
    c->last_timed = timing;
    if (dirty_out) {
        CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *dirty_out = c->h_st->K;
    }
    return CRUM_OK;
}

// ---------------------------------------------------------------------------
// A1-A3 into a device image: detect, compact (+ table, header fields),
// gather (+ commit), CRC (+ tail, header).  Fully stream-ordered.
// ---------------------------------------------------------------------------
int crum_checkpoint_gather_device(crum_ctx *ctx, void *dev_image, uint64_t capacity, void *stream,
                                  uint32_t flags, crum_report *rep) {
    NvtxRange nvtx_("crum_checkpoint_gather_device");
    ENTER(ctx);
    NOT_IN_SESSION(c);
    if (!dev_image || (flags & ~(CRUM_FULL | CRUM_COMPRESS)) || (reinterpret_cast<uintptr_t>(dev_image) & 255)) {
        set_detail("bad device image pointer (must be 256-byte aligned) or flags");
        return CRUM_E_INVAL;
    }
    if (!rep) {
        uint64_t need;
        crum_image_required_bytes(c, UINT64_MAX, &need);
        if (capacity < need) {
            set_detail("asynchronous device gather needs capacity >= %llu", (unsigned long long)need);
            return CRUM_E_CAPACITY;
        }
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool full = flags & CRUM_FULL;
    const bool timing = rep != nullptr || c->timing_cfg;
    uint8_t *img = static_cast<uint8_t *>(dev_image);
    int st;
    uint64_t worst = 0;
    crum_image_required_bytes(c, UINT64_MAX, &worst);
    if (flags & CRUM_COMPRESS) return gather_z(c, s, img, nullptr, capacity, full, timing, rep);
    if (!rep && c->graphs_on) {
        // asynchronous call: replay the captured sequence (the one-launch small
        // path, the single pass, or the multi-kernel sequence: chosen and
        // keyed inside; one launch instead of ~8 API calls)
        if ((st = gather_dev_graph(c, s, img, capacity, flags, timing)) != CRUM_E_BUSY) {
            if (st == CRUM_OK) {
                c->last_timed = timing;
                c->last_path = 0;
            }
            return st;
        }
        // capture not possible here: enqueue directly
    }
    const bool small = use_small(c, full, capacity, worst);
    if (small || use_fused(c, full, capacity, worst)) {
        // single pass: detect + compact + gather + commit in one kernel (the
        // small path also writes the metadata; the single-pass kernel is
        // followed by the metadata CRC / tail / header)
        st = small ? enqueue_small(c, s, img, capacity, timing) : enqueue_fused(c, s, img, capacity, timing);
        if (st) return st;
        c->last_kind = kLastDevFused;
        c->last_small = small;
        c->last_path = 0;
        c->last_timed = timing;
        if (rep) {
            CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            memset(rep, 0, sizeof *rep);
            fill_report(c, *c->h_st, rep);
            fill_times(c, *c->h_st, rep);
        }
        return CRUM_OK;
    }
    if ((st = enqueue_gather_dev(c, s, img, capacity, full, timing))) return st;
    c->last_path = 0;
    c->last_kind = kLastDevGather;
    c->last_timed = timing;
    if (rep) {
        CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const DevStats h = *c->h_st;
        memset(rep, 0, sizeof *rep);
        fill_report(c, h, rep);
        fill_times(c, h, rep);
        if (h.status == kStCapacity) {
            set_detail("image needs %llu bytes, capacity %llu", (unsigned long long)h.image_bytes,
                       (unsigned long long)capacity);
            return CRUM_E_CAPACITY;
        }
    }
    return CRUM_OK;
}

// ---------------------------------------------------------------------------
// A1-A4 into a pinned host image.  The page space is cut into ranges; for
// each range detect + compact run on the caller's stream, the host reads the
// range's running totals and immediately enqueues gathers (side stream, into
// a ring of device chunks) and D2H copies (copy stream) of its payload, so
// the host-link transfer of range c overlaps the detection of range c+1.
// If the image cannot hold a worst-case image, the call first waits for all
// ranges and checks capacity before committing anything.
// ---------------------------------------------------------------------------
int crum_checkpoint_gather(crum_ctx *ctx, crum_image *img, void *stream, uint32_t flags, crum_report *rep) {
    NvtxRange nvtx_("crum_checkpoint_gather");
    ENTER(ctx);
    NOT_IN_SESSION(c);
    if (!img || (flags & ~(CRUM_FULL | CRUM_COMPRESS))) {
        set_detail("null image or bad flags");
        return CRUM_E_INVAL;
    }
    if (img->busy.load() || img->sessions) {
        set_detail(img->sessions ? "a lazy restore session reads this image"
                                 : "image is being persisted (alternate two images)");
        return CRUM_E_BUSY;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool full = flags & CRUM_FULL;
    if (flags & CRUM_COMPRESS) return gather_z(c, s, nullptr, img, img->cap, full, true, rep);
    c->last_path = 0;
    uint64_t worst;
    crum_image_required_bytes(c, UINT64_MAX, &worst);
    const bool graphs_on = c->graphs_on;
    if (worst <= std::min(kSmallImage, c->chunk) && img->cap >= worst) {
        // small footprint: latency-bound, so run the device sequence (a replayed
        // graph) with the image's mapped address as the destination -- the
        // kernels' stores cross the host link directly, no staging, no copies
        void *dimg = nullptr;
        CK(cudaHostGetDevicePointer(&dimg, img->host, 0));
        uint8_t *d = static_cast<uint8_t *>(dimg);
        int st = graphs_on ? gather_dev_graph(c, s, d, img->cap, flags, true) : CRUM_E_BUSY;
        if (st == CRUM_E_BUSY) {
            const bool small = use_small(c, full, img->cap, worst);
            const bool fused = !small && use_fused(c, full, img->cap, worst);
            st = small ? enqueue_small(c, s, d, img->cap, true)
                 : fused ? enqueue_fused(c, s, d, img->cap, true)
                         : enqueue_gather_dev(c, s, d, img->cap, full, true);
            c->last_kind = (small || fused) ? kLastDevFused : kLastDevGather;
            c->last_small = small;
        }
        if (st) return st;  // (gather_dev_graph set last_kind)
        c->last_path = 0;
        c->last_timed = true;
        // every small-footprint sequence's last kernel stores the final stats
        // into the mapped h_st: no copy, only the wait
        CK(cudaStreamSynchronize(s));
        const DevStats h = *c->h_st;
        img->len = h.image_bytes;
        if (rep) {
            memset(rep, 0, sizeof *rep);
            fill_report(c, h, rep);
            fill_times(c, h, rep);
        }
        return CRUM_OK;
    }
    int st = ensure_ring(c);
    if (st) return st;
    // An image that holds a worst-case image cannot overflow: gathers commit
    // as they copy.  A smaller image (the usual case at large footprints: a
    // worst-case image is as large as the footprint) still streams range by
    // range, but its gathers only copy; the commit runs as one more pass after
    // the final range's metadata shows the image fits, so a CAPACITY error
    // commits nothing (crum.h).  That pass re-reads the dirty pages of
    // compare-mode regions once (KP of HBM reads, overlapped with the copy-out).
    const bool deferred = img->cap < worst;
    // Ranges exist to overlap the copy-out of range c with the detection of
    // range c + 1; when the previous checkpoint's payload was small (the copy
    // is short) one range avoids a host wait per range (C2 at 0 % dirty: 10
    // waits of the host on range events were half the step).  A heuristic on
    // the mapped stats of the previous call only: the image is the same.
    const uint64_t prev_payload = *reinterpret_cast<volatile const uint64_t *>(&c->h_st->payload_bytes);
    const bool one_range = prev_payload <= kOneRangePayload;
    // ... and where nothing can overflow, mapped stores with no host wait at
    // all (a one-range kernel sequence stores after the detection, so only
    // very small payloads take it; the single pass overlaps the two)
    const bool mapped_ok = !deferred && !full && c->gathers_since_rebuild > 0 && c->mapped_cfg;
    if (mapped_ok && one_range)
        return gather_mapped(c, s, img, c->fused_ok && prev_payload > kMappedSerialPayload,
                             prev_payload > kMappedOneRange, rep);
    // the single pass also up to kMappedFusedPayload: its stores overlap the
    // detection, where the ring pipeline pays a host wait per range
    if (mapped_ok && c->fused_ok && prev_payload <= kMappedFusedPayload)
        return gather_mapped(c, s, img, true, false, rep);
    const uint32_t nr = one_range ? 1u : (uint32_t)c->ranges.size();
    auto range_at = [&](uint32_t ci) -> const Range & { return one_range ? c->all : c->ranges[ci]; };
    const uint64_t poff = payload_offset_for(c->regs.size());
    void *dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, img->host, 0));
    uint8_t *dimg = static_cast<uint8_t *>(dp);  // the image's mapped address (metadata)
    CK(cudaEventRecord(c->ev_t[0], s));
    CK(cudaMemsetAsync(c->d_rb, 0, sizeof(RangeTotals), s));
    // detect + compact of range ci on the caller's stream; after the last range
    // the metadata CRC + tail go into d_meta (tail after the head [0, poff))
    uint32_t enq = 0;
    auto enqueue_range = [&](uint32_t ci) -> int {
        const Range &rg = range_at(ci);
        enqueue_detect(c, s, rg, full);
        // the final compaction checks the image's capacity: a CAPACITY status
        // stops the CRC kernel before it writes anything into the image
        enqueue_compact(c, s, compact_args(c, rg, ci, ci == 0, ci + 1 == nr, full, img->cap, c->d_meta));
        CK_LAUNCH();
        CK(cudaEventRecord(c->ev_range[ci], s));  // h_rb[ci + 1] written by the kernel (mapped)
        if (c->trace) CK(cudaEventRecord(c->ev_trace[3 * ci], s));
        if (ci + 1 == nr) {
            CK(cudaEventRecord(c->ev_t[1], s));
            // header, table, padding and tail straight into the pinned image
            // through its mapped address (no metadata copies, no host wait at
            // the end); the final stats into mapped memory
            CrcArgs cra = crc_args(c, c->d_meta, nullptr);
            cra.out = dimg;
            launch_crc_meta(launch_of(c, s), cra, crc_max_len(c));
            CK_LAUNCH();
            CK(cudaEventRecord(c->ev_meta, s));  // h_st written by the CRC kernel (mapped)
        }
        return CRUM_OK;
    };
    // keep the GPU kAhead ranges ahead of the host
    constexpr uint32_t kAhead = 2;
    while (enq < nr && enq < kAhead)
        if ((st = enqueue_range(enq++))) return st;
    // payload: per range, gathers into the ring + D2H
    Launch G = launch_of(c, c->gstream);
    const uint64_t upc = c->chunk >> kSegLog2;
    uint64_t chunk_idx = 0;
    bool copy_started = false, overflow = false;
    c->h_rb[0] = RangeTotals{0, 0};
    for (uint32_t ci = 0; ci < nr; ++ci) {
        while (enq < nr && enq <= ci + kAhead)
            if ((st = enqueue_range(enq++))) return st;
        CK(cudaEventSynchronize(c->ev_range[ci]));
        const uint64_t U0 = c->h_rb[ci].units, U1 = c->h_rb[ci + 1].units;
        // the image so far (payload of ranges <= ci, and the ids / hashes of
        // their pages) already exceeds the capacity: stop copying, keep
        // compacting to learn the required size
        if (deferred && !overflow &&
            poff + (U1 << kSegLog2) + tail_bytes_for(c->h_rb[ci + 1].k, c->any_hash) > img->cap)
            overflow = true;
        if (overflow) continue;
        if (U1 > U0) CK(cudaStreamWaitEvent(c->gstream, c->ev_range[ci], 0));
        for (uint64_t u0 = U0; u0 < U1; u0 += upc, ++chunk_idx) {
            const uint64_t u1 = std::min(U1, u0 + upc);
            const int slot = (int)(chunk_idx % kRing);
            if (chunk_idx >= (uint64_t)kRing) CK(cudaStreamWaitEvent(c->gstream, c->ev_copy[slot], 0));
            GatherArgs ga = gather_args(c, ci, c->d_ring[slot], u0, false, u0, u1);
            ga.no_commit = deferred ? 1 : 0;
            launch_gather(G, ga, u1 - u0);
            CK_LAUNCH();
            CK(cudaEventRecord(c->ev_gather[slot], c->gstream));
            CK(cudaStreamWaitEvent(c->copy, c->ev_gather[slot], 0));
            if (!copy_started) {
                CK(cudaEventRecord(c->ev_t[4], c->copy));
                copy_started = true;
            }
            CK(cudaMemcpyAsync(img->host + poff + (u0 << kSegLog2), c->d_ring[slot], (u1 - u0) << kSegLog2,
                               cudaMemcpyDeviceToHost, c->copy));
            CK(cudaEventRecord(c->ev_copy[slot], c->copy));
        }
        if (c->trace) {
            CK(cudaEventRecord(c->ev_trace[3 * ci + 1], c->gstream));
            CK(cudaEventRecord(c->ev_trace[3 * ci + 2], c->copy));
        }
    }
    if (deferred) {
        CK(cudaEventSynchronize(c->ev_meta));
        if (overflow || c->h_st->image_bytes > img->cap) {
            CK(cudaStreamSynchronize(c->gstream));
            CK(cudaStreamSynchronize(c->copy));
            CK(cudaStreamSynchronize(s));
            if (rep) {
                memset(rep, 0, sizeof *rep);
                fill_report(c, *c->h_st, rep);
            }
            set_detail("image needs %llu bytes, capacity %llu", (unsigned long long)c->h_st->image_bytes,
                       (unsigned long long)img->cap);
            return CRUM_E_CAPACITY;
        }
        // the image fits: commit every listed page (mirror / table / force),
        // range by range, on the gather stream behind the copies' gathers
        CK(cudaStreamWaitEvent(c->gstream, c->ev_meta, 0));
        for (uint32_t ci = 0; ci < nr; ++ci) {
            const uint64_t U0 = c->h_rb[ci].units, U1 = c->h_rb[ci + 1].units;
            if (U1 > U0) {
                launch_gather(G, gather_args(c, ci, nullptr, 0, false, U0, U1), U1 - U0);
                CK_LAUNCH();
            }
        }
    }
    // the metadata went in through the mapped address (CRC kernel on s)
    if (!copy_started) CK(cudaEventRecord(c->ev_t[4], c->copy));
    CK(cudaStreamWaitEvent(c->copy, c->ev_meta, 0));
    CK(cudaEventRecord(c->ev_t[5], c->copy));
    CK(cudaEventRecord(c->ev_t[3], c->gstream));
    CK(cudaStreamSynchronize(c->gstream));
    CK(cudaStreamSynchronize(c->copy));
    CK(cudaStreamSynchronize(s));
    const DevStats h = *c->h_st;
    CK(cudaEventRecord(c->ev_done, s));
    ++c->gathers_since_rebuild;
    c->last_kind = kLastHostGather;
    c->last_timed = true;
    img->len = h.image_bytes;
    if (c->trace) {
        fprintf(stderr, "[crum trace] gather: %u ranges, K=%llu, payload=%llu B, t_detect_all=%.3f ms\n", nr,
                (unsigned long long)h.K, (unsigned long long)h.payload_bytes, ev_ms(c->ev_t[0], c->ev_t[1]));
        for (uint32_t ci = 0; ci < nr; ++ci)
            fprintf(stderr, "[crum trace]  range %2u pages [%llu,%llu) units %llu: compacted %.3f  gathered %.3f  "
                            "copied %.3f ms\n",
                    ci, (unsigned long long)range_at(ci).p_lo, (unsigned long long)range_at(ci).p_hi,
                    (unsigned long long)(c->h_rb[ci + 1].units - c->h_rb[ci].units),
                    ev_ms(c->ev_t[0], c->ev_trace[3 * ci]), ev_ms(c->ev_t[0], c->ev_trace[3 * ci + 1]),
                    ev_ms(c->ev_t[0], c->ev_trace[3 * ci + 2]));
        fprintf(stderr, "[crum trace]  meta copied %.3f ms\n", ev_ms(c->ev_t[0], c->ev_t[5]));
    }
    if (rep) {
        memset(rep, 0, sizeof *rep);
        fill_report(c, h, rep);
        fill_times(c, h, rep);
    }
    return CRUM_OK;
}

// ---------------------------------------------------------------------------
// A6: restore scatter
// ---------------------------------------------------------------------------
namespace {

struct ParsedImage {
    uint32_t flags, R;
    uint64_t K, poff, payload, ids_off, image;
    uint64_t upayload = 0;  // payload bytes before compression (= payload unless flag bit2)
    std::vector<RegStat> rs;
    std::vector<DevRegion> tregs;
};

// Host-side checks of the header (every CORRUPT condition that needs no
// device data).
int parse_header(const uint8_t *hdr, uint64_t len, ParsedImage &p) {
    if (len < 64 || memcmp(hdr, "CRUM", 4) != 0) return CRUM_E_CORRUPT;
    if (crc32_host(hdr, 60) != rd32(hdr + 60)) return CRUM_E_CORRUPT;
    const uint32_t version = rd32(hdr + 4);
    p.flags = rd32(hdr + 8);
    p.R = rd32(hdr + 12);
    p.K = rd64(hdr + 16);
    p.poff = rd64(hdr + 24);
    p.payload = rd64(hdr + 32);
    p.ids_off = rd64(hdr + 40);
    p.image = rd64(hdr + 48);
    if (version != 1 || (p.flags & ~7u)) return CRUM_E_CORRUPT;
    if (p.K > kMaxTotalPages || p.R > 0x7fffffffu) return CRUM_E_CORRUPT;
    if (p.poff != payload_offset_for(p.R) || p.payload > (1ull << 62) || p.ids_off != p.poff + p.payload)
        return CRUM_E_CORRUPT;
    const uint64_t tail = tail_bytes_for(p.K, p.flags & 2u);
    if (!(p.flags & 4u) && p.image != p.ids_off + tail) return CRUM_E_CORRUPT;
    // compressed: the exact length needs the unit count (parse_table)
    if ((p.flags & 4u) && ((p.payload & (kSegBytes - 1)) || p.image < p.ids_off + tail ||
                           p.image - p.ids_off - tail > (1ull << 62)))
        return CRUM_E_CORRUPT;
    if (len < p.image) return CRUM_E_CORRUPT;
    return CRUM_OK;
}

int parse_table(const uint8_t *tab, ParsedImage &p) {
    p.rs.assign(p.R, RegStat{});
    p.tregs.assign(p.R, DevRegion{});
    uint64_t sum = 0, pay = 0;
    bool any_hash = false;
    for (uint32_t k = 0; k < p.R; ++k) {
        const uint8_t *e = tab + 48ull * k;
        const uint32_t mode = rd32(e + 4);
        const uint64_t bytes = rd64(e + 8), ps = rd64(e + 16), np = rd64(e + 24), nd = rd64(e + 32),
                       first = rd64(e + 40);
        if (mode > 2 || ps < 4096 || ps > (2u << 20) || (ps & (ps - 1)) || bytes == 0) return CRUM_E_CORRUPT;
        if (np != bytes / ps + (bytes % ps != 0) || nd > np || first != sum) return CRUM_E_CORRUPT;
        if ((p.flags & 1u) && nd != np) return CRUM_E_CORRUPT;
        if (mode == 1) any_hash = true;
        p.rs[k].first = first;
        p.rs[k].n_dirty = nd;
        p.rs[k].payload_base = pay;
        p.rs[k].unit_base = pay >> kSegLog2;
        DevRegion &d = p.tregs[k];
        d.bytes = bytes;
        d.n_pages = np;
        d.log2p = (uint32_t)__builtin_ctzll(ps);
        d.mode = mode;
        d.id = rd32(e);
        sum += nd;
        pay += nd * ps;
    }
    const bool z = (p.flags & 4u) != 0;
    if (sum != p.K || (!z && pay != p.payload) || any_hash != ((p.flags & 2u) != 0)) return CRUM_E_CORRUPT;
    if (z && p.image != p.ids_off + tail_bytes_for(p.K, p.flags & 2u) + round_up(2 * (pay >> kSegLog2), 8))
        return CRUM_E_CORRUPT;
    p.upayload = pay;
    return CRUM_OK;
}

int check_live(crum_ctx *c, const uint8_t *tab, const ParsedImage &p) {
    if (p.R != c->regs.size()) return CRUM_E_MISMATCH;
    for (uint32_t k = 0; k < p.R; ++k) {
        const uint8_t *e = tab + 48ull * k;
        const HostRegion &h = c->regs[k];
        if (rd32(e) != h.id || rd32(e + 4) != h.mode || rd64(e + 8) != h.bytes || rd64(e + 16) != h.page_size ||
            rd64(e + 24) != h.n_pages)
            return CRUM_E_MISMATCH;
    }
    return CRUM_OK;
}

// Common restore body.  host_img != nullptr: image in pinned host memory
// (payload goes H2D in chunks); else dev_img holds the whole image.
// Validated restore: the parsed image, its metadata on the device, and the
// payload's device address when it is already device-visible.
struct PreparedRestore {
    ParsedImage p;
    std::vector<uint8_t> tab;
    const uint32_t *d_ids = nullptr;
    const uint64_t *d_hashes = nullptr;
    const uint8_t *payload_dev = nullptr;
    uint8_t *d_payload_tmp = nullptr;  // decoded / CRUM_VERIFY staging of the payload
    bool tmp_owned = false;            // the caller frees d_payload_tmp (else it is c->d_rtmp)
    bool z_lazy = false;               // compressed, checked but not decoded (lazy session)
    const uint8_t *zsrc = nullptr;     // its encoded payload, device-visible (mapped)
    DevStats hst{};                    // K, dirty bytes, runs of the image
};

// Every check of a restore (header, table, metadata CRC, ids, live set,
// CRUM_VERIFY) before anything is written.  On return the table and tail
// are in c->d_meta (host image) and the region stats in c->d_rs / c->d_st.
int prepare_restore(crum_ctx *c, const uint8_t *host_img, const uint8_t *dev_img, uint64_t len, cudaStream_t s,
                    uint32_t flags, bool timing, PreparedRestore &pr, bool cached, bool lazy_z = false) {
    // payload staging: the context's grow-only buffer, or one owned by the caller
    auto tmp_alloc = [&](uint8_t **q, uint64_t bytes) -> int {
        if (!cached) return dev_alloc(c, q, bytes);
        int e = grow(c, &c->d_rtmp, &c->rtmp_cap, bytes);
        *q = c->d_rtmp;
        return e;
    };
    auto tmp_free = [&](uint8_t *q) {
        if (!cached && q) cudaFree(q);
    };
    pr.tmp_owned = !cached;
    ParsedImage &p = pr.p;
    uint8_t hdr[64];
    if (len < 64) {
        set_detail("image shorter than its header");
        return CRUM_E_CORRUPT;
    }
    if (host_img) {
        memcpy(hdr, host_img, 64);
    } else {
        CK(cudaMemcpyAsync(hdr, dev_img, 64, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    int st = parse_header(hdr, len, p);
    if (st) {
        set_detail("bad image header");
        return st;
    }
    std::vector<uint8_t> &tab = pr.tab;
    tab.resize(48ull * p.R);
    if (p.R) {
        if (host_img) {
            memcpy(tab.data(), host_img + 64, tab.size());
        } else {
            CK(cudaMemcpyAsync(tab.data(), dev_img + 64, tab.size(), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    if ((st = parse_table(tab.data(), p))) {
        set_detail("bad image region table");
        return st;
    }
    const bool hh = (p.flags & 2u) != 0;
    const uint64_t tail_len = p.image - p.ids_off;
    const uint64_t tab_len = 48ull * p.R;
    if (timing) CK(cudaEventRecord(c->ev_t[0], s));
    // table + tail on the device
    const uint8_t *d_table, *d_tail;
    if (host_img) {
        const uint64_t need = round_up(tab_len, 16) + tail_len + 16;
        if (need > c->meta_cap) {
            dev_free(c->d_meta);
            c->meta_cap = 0;
            if ((st = dev_alloc(c, &c->d_meta, need))) return st;
            c->meta_cap = need;
        }
        if (tab_len) CK(cudaMemcpyAsync(c->d_meta, host_img + 64, tab_len, cudaMemcpyHostToDevice, s));
        if (tail_len)
            CK(cudaMemcpyAsync(c->d_meta + round_up(tab_len, 16), host_img + p.ids_off, tail_len,
                               cudaMemcpyHostToDevice, s));
        d_table = c->d_meta;
        d_tail = c->d_meta + round_up(tab_len, 16);
    } else {
        d_table = dev_img + 64;
        d_tail = dev_img + p.ids_off;
    }
    const uint32_t *d_ids = reinterpret_cast<const uint32_t *>(d_tail);
    const uint64_t *d_hashes = hh ? reinterpret_cast<const uint64_t *>(d_tail + round_up(4 * p.K, 8)) : nullptr;
    if (p.R + 1 > c->rs_cap) {
        dev_free(c->d_rs);
        c->rs_cap = 0;
        if ((st = dev_alloc(c, &c->d_rs, sizeof(RegStat) * (p.R + 1)))) return st;
        c->rs_cap = p.R + 1;
    }
    if (p.R > c->tregs_cap) {
        dev_free(c->d_tregs);
        c->tregs_cap = 0;
        if ((st = dev_alloc(c, &c->d_tregs, sizeof(DevRegion) * p.R))) return st;
        c->tregs_cap = p.R;
    }
    DevStats hs{};
    hs.K = p.K;
    hs.poff = p.poff;
    hs.payload_bytes = p.payload;
    hs.ids_off = p.ids_off;
    hs.image_bytes = p.image;
    hs.total_units = p.upayload >> kSegLog2;
    hs.img_flags = p.flags;
    hs.n_regions = p.R;
    *c->h_st = hs;
    CK(cudaMemcpyAsync(c->d_st, c->h_st, sizeof(DevStats), cudaMemcpyHostToDevice, s));
    if (p.R) {
        CK(cudaMemcpyAsync(c->d_rs, p.rs.data(), sizeof(RegStat) * p.R, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(c->d_tregs, p.tregs.data(), sizeof(DevRegion) * p.R, cudaMemcpyHostToDevice, s));
    }
    Launch L = launch_of(c, s);
    if (tab_len + tail_len) launch_crc_check(L, d_table, tab_len, d_tail, tail_len, c->d_st, crc_tables().x2n);
    launch_restore_validate(L, c->d_tregs, p.R, c->d_rs, d_ids, d_hashes, p.K, c->d_st);
    // compressed: every unit size <= 4096, sizes summing to the payload (readings Z2-Z3)
    const bool zimg = (p.flags & 4u) != 0;
    const uint64_t zunits = p.upayload >> kSegLog2;
    const uint16_t *d_zsz = reinterpret_cast<const uint16_t *>(d_tail + tail_bytes_for(p.K, hh));
    if (zimg) {
        if ((st = ensure_z(c, zunits))) return st;
        launch_zscan(L, d_zsz, c->d_st, c->d_zloc, c->d_zblk, zunits);
    }
    CK_LAUNCH();
    CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    {
        const DevStats h = *c->h_st;
        const uint32_t meta_crc = (tab_len + tail_len == 0) ? 0u : (h.crc_acc ^ 0xffffffffu);
        if (meta_crc != rd32(hdr + 56) || h.status != kStOk) {
            set_detail(meta_crc != rd32(hdr + 56) ? "metadata CRC mismatch" : "bad page id list");
            return CRUM_E_CORRUPT;
        }
        pr.hst = h;
    }
    if ((st = check_live(c, tab.data(), p))) {
        set_detail("image region table does not match the registered regions");
        return st;
    }
    uint8_t *d_payload_tmp = nullptr;
    const uint8_t *payload_dev = dev_img ? dev_img + p.poff : nullptr;
    // compressed: decode every unit into device memory first (a unit that is
    // not a valid encoding is CORRUPT); a pinned image's encoded payload
    // crosses the link once (copy engine), then decodes from HBM
    if (zimg && lazy_z && host_img && !(flags & CRUM_VERIFY)) {
        // lazy session: validate every unit now by decoding it in place
        // through the mapped address without storing the result (the same
        // CORRUPT verdict as a full decode), decode windows on demand later
        void *dp = nullptr;
        CK(cudaHostGetDevicePointer(&dp, const_cast<uint8_t *>(host_img), 0));
        pr.zsrc = static_cast<const uint8_t *>(dp) + p.poff;
        pr.z_lazy = true;
        launch_zdecode(L, pr.zsrc, d_zsz, c->d_zloc, c->d_zblk, c->d_st, nullptr, zunits);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (c->h_st->status != kStOk) {
            set_detail("compressed unit that is not a valid encoding");
            return CRUM_E_CORRUPT;
        }
    } else if (zimg) {
        const uint8_t *src = payload_dev;
        if (host_img) {
            if ((st = grow(c, &c->d_renc, &c->renc_cap, p.payload))) return st;
            CK(cudaMemcpyAsync(c->d_renc, host_img + p.poff, p.payload, cudaMemcpyHostToDevice, s));
            src = c->d_renc;
        }
        if ((st = tmp_alloc(&d_payload_tmp, p.upayload))) return st;
        launch_zdecode(L, src, d_zsz, c->d_zloc, c->d_zblk, c->d_st, d_payload_tmp, zunits);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (c->h_st->status != kStOk) {
            tmp_free(d_payload_tmp);
            set_detail("compressed unit that is not a valid encoding");
            return CRUM_E_CORRUPT;
        }
        payload_dev = d_payload_tmp;
    }
    // CRUM_VERIFY: hash every hash-mode slot before writing anything
    if ((flags & CRUM_VERIFY) && c->any_hash && p.K) {
        if (!payload_dev) {
            if ((st = tmp_alloc(&d_payload_tmp, p.upayload))) return st;
            CK(cudaMemcpyAsync(d_payload_tmp, host_img + p.poff, p.upayload, cudaMemcpyHostToDevice, s));
            payload_dev = d_payload_tmp;
        }
        launch_verify_hash(L, c->d_regs, p.R, c->d_rs, d_hashes, payload_dev, p.K, c->d_st);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (c->h_st->status != kStOk) {
            tmp_free(d_payload_tmp);
            set_detail("CRUM_VERIFY: a hash-mode slot does not match its listed hash");
            return CRUM_E_CORRUPT;
        }
    }
    pr.d_ids = d_ids;
    pr.d_hashes = d_hashes;
    pr.payload_dev = payload_dev;
    pr.d_payload_tmp = d_payload_tmp;
    return CRUM_OK;
}

int restore_common(crum_ctx *c, const uint8_t *host_img, const uint8_t *dev_img, uint64_t len, cudaStream_t s,
                   uint32_t flags, crum_report *rep) {
    const bool timing = rep != nullptr || c->timing_cfg;
    PreparedRestore pr;
    int st = prepare_restore(c, host_img, dev_img, len, s, flags, timing, pr, true);
    if (st) return st;
    const ParsedImage &p = pr.p;
    const uint32_t *d_ids = pr.d_ids;
    const uint64_t *d_hashes = pr.d_hashes;
    const uint8_t *payload_dev = pr.payload_dev;
    uint8_t *d_payload_tmp = pr.d_payload_tmp;
    Launch L = launch_of(c, s);
    if (timing) CK(cudaEventRecord(c->ev_t[1], s));
    const uint64_t units = p.upayload >> kSegLog2;
    ScatterArgs sa{};
    sa.regs = c->d_regs;
    sa.R = p.R;
    sa.rs = c->d_rs;
    sa.ids = d_ids;
    sa.hashes = d_hashes;
    sa.st = c->d_st;
    sa.force = c->d_force;
    if (payload_dev) {
        sa.src = payload_dev;
        sa.src_unit0 = 0;
        sa.u_lo = 0;
        sa.u_hi = units;
        launch_scatter(L, sa);
        CK_LAUNCH();
        if (timing) {
            CK(cudaEventRecord(c->ev_t[4], s));
            CK(cudaEventRecord(c->ev_t[5], s));
        }
    } else {
        if ((st = ensure_ring(c))) return st;
        const uint64_t upc = c->chunk >> kSegLog2;
        uint64_t ci = 0;
        CK(cudaEventRecord(c->ev_meta, s));
        CK(cudaStreamWaitEvent(c->copy, c->ev_meta, 0));
        if (timing) CK(cudaEventRecord(c->ev_t[4], c->copy));
        for (uint64_t u0 = 0; u0 < units; u0 += upc, ++ci) {
            const uint64_t u1 = std::min(units, u0 + upc);
            const int slot = (int)(ci % kRing);
            if (ci >= (uint64_t)kRing) CK(cudaStreamWaitEvent(c->copy, c->ev_gather[slot], 0));
            CK(cudaMemcpyAsync(c->d_ring[slot], host_img + p.poff + (u0 << kSegLog2), (u1 - u0) << kSegLog2,
                               cudaMemcpyHostToDevice, c->copy));
            CK(cudaEventRecord(c->ev_copy[slot], c->copy));
            CK(cudaStreamWaitEvent(s, c->ev_copy[slot], 0));
            sa.src = c->d_ring[slot];
            sa.src_unit0 = u0;
            sa.u_lo = u0;
            sa.u_hi = u1;
            launch_scatter(L, sa);
            CK_LAUNCH();
            CK(cudaEventRecord(c->ev_gather[slot], s));
        }
        if (timing) CK(cudaEventRecord(c->ev_t[5], c->copy));
    }
    if (timing) CK(cudaEventRecord(c->ev_t[3], s));
    CK(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamSynchronize(c->copy));
    if (d_payload_tmp && pr.tmp_owned) cudaFree(d_payload_tmp);
    CK(cudaEventRecord(c->ev_done, s));
    c->last_kind = kLastRestore;
    c->last_path = 0;
    c->last_timed = timing;
    if (rep) {
        memset(rep, 0, sizeof *rep);
        fill_report(c, *c->h_st, rep);
        rep->image_bytes = p.image;
        fill_times(c, *c->h_st, rep);
    }
    return CRUM_OK;
}

}  // namespace

int crum_restore_scatter(crum_ctx *ctx, const crum_image *img, void *stream, uint32_t flags, crum_report *rep) {
    NvtxRange nvtx_("crum_restore_scatter");
    ENTER(ctx);
    NOT_IN_SESSION(c);
    if (!img || (flags & ~CRUM_VERIFY)) {
        set_detail("null image or bad flags");
        return CRUM_E_INVAL;
    }
    // reading an image that is being persisted is safe (the writer only reads)
    return restore_common(c, img->host, nullptr, img->len, static_cast<cudaStream_t>(stream), flags, rep);
}

int crum_restore_scatter_device(crum_ctx *ctx, const void *dev_image, uint64_t len, void *stream, uint32_t flags,
                                crum_report *rep) {
    NvtxRange nvtx_("crum_restore_scatter_device");
    ENTER(ctx);
    NOT_IN_SESSION(c);
    if (!dev_image || (flags & ~CRUM_VERIFY) || (reinterpret_cast<uintptr_t>(dev_image) & 255)) {
        set_detail("bad device image pointer (must be 256-byte aligned) or flags");
        return CRUM_E_INVAL;
    }
    return restore_common(c, nullptr, static_cast<const uint8_t *>(dev_image), len,
                          static_cast<cudaStream_t>(stream), flags, rep);
}

// ---------------------------------------------------------------------------
// Lazy restore with exponential prefetch (sec. 4.2 heuristic, PAPER.md:783-793;
// SURVEY.md sec. 8(f) #3).  begin validates everything (as crum_restore_scatter)
// and writes nothing; every fetch is the analog of a read fault on a page of a
// region: it restores the window the heuristic names, reading the image's
// slots straight from the mapped pinned image (zero-copy) or, after
// CRUM_VERIFY, from the verified device copy; end restores what is left.
// ---------------------------------------------------------------------------
struct crum_restore_session {
    crum_ctx *c = nullptr;
    crum_image *img = nullptr;
    ParsedImage p;
    std::vector<uint8_t> tab;
    const uint8_t *payload_src = nullptr;   // device-visible payload
    uint8_t *d_payload_tmp = nullptr;       // owned (CRUM_VERIFY copy)
    uint8_t *d_tail = nullptr;              // owned copy of ids (+ hashes)
    RegStat *d_rs = nullptr;
    DevStats *d_st = nullptr;
    uint8_t *d_done = nullptr;              // per slot: written
    std::vector<uint8_t> covered;           // per global page: present (fetched)
    std::vector<uint64_t> window;           // per region: pages the next fault reads
    DevStats hst{};
    uint64_t restored = 0, covered_pages = 0;
    // compressed image restored lazily: windows are decoded on demand from
    // the pinned image (mapped) into pool buffers, unit offsets from the ctx scan
    bool z_lazy = false;
    const uint8_t *zsrc = nullptr;
};

namespace {
constexpr uint64_t kSmallRegionPages = 8;  // DESIGN.md reading: "small" = at most 8 pages

void session_free(crum_restore_session *ss) {
    dev_free(ss->d_payload_tmp);
    dev_free(ss->d_tail);
    dev_free(ss->d_rs);
    dev_free(ss->d_st);
    dev_free(ss->d_done);
}

// Scatter slots [klo, khi) of table entry k (all of them uncovered until now).
int session_scatter_slots(crum_restore_session *ss, uint32_t k, uint64_t klo, uint64_t khi, cudaStream_t s) {
    crum_ctx *c = ss->c;
    const RegStat &r = ss->p.rs[k];
    const uint32_t sh = c->regs[k].log2p - kSegLog2;
    ScatterArgs sa{};
    sa.regs = c->d_regs;
    sa.R = ss->p.R;
    sa.rs = ss->d_rs;
    sa.ids = reinterpret_cast<const uint32_t *>(ss->d_tail);
    sa.hashes = (ss->p.flags & 2u) ? reinterpret_cast<const uint64_t *>(ss->d_tail + round_up(4 * ss->p.K, 8))
                                   : nullptr;
    sa.st = ss->d_st;
    sa.src = ss->payload_src;
    sa.src_unit0 = 0;
    sa.force = c->d_force;
    sa.u_lo = r.unit_base + ((klo - r.first) << sh);
    sa.u_hi = r.unit_base + ((khi - r.first) << sh);
    sa.mark = ss->d_done;
    if (ss->z_lazy) {
        // the window's encoded bytes cross the link once (wide zero-copy reads
        // into a pool buffer), then decode from HBM into another
        const uint64_t nu = sa.u_hi - sa.u_lo;
        // window buffers from the stream-ordered pool: no device-wide
        // synchronisation, memory reused across faults
        const uint64_t need = nu << kSegLog2;
        uint8_t *win = nullptr, *enc = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void **>(&win), need, s));
        CK(cudaMallocAsync(reinterpret_cast<void **>(&enc), need + 64, s));  // + word alignment slack
        const uint16_t *zsz = reinterpret_cast<const uint16_t *>(
            ss->d_tail + tail_bytes_for(ss->p.K, (ss->p.flags & 2u) != 0));
        const Launch L = launch_of(c, s);
        launch_zfetch(L, ss->zsrc, zsz, c->d_zloc, c->d_zblk, sa.u_lo, sa.u_hi, enc);
        launch_zdecode(L, enc, zsz, c->d_zloc, c->d_zblk, ss->d_st, win, nu, sa.u_lo, 1);
        sa.src = win;
        sa.src_unit0 = sa.u_lo;
        launch_scatter(L, sa);
        CK_LAUNCH();
        CK(cudaFreeAsync(enc, s));
        CK(cudaFreeAsync(win, s));
        return CRUM_OK;
    }
    launch_scatter(launch_of(c, s), sa);
    CK_LAUNCH();
    return CRUM_OK;
}
}  // namespace

int crum_restore_begin(crum_ctx *ctx, crum_image *img, void *stream, uint32_t flags, crum_restore_session **out) {
    NvtxRange nvtx_("crum_restore_begin");
    ENTER(ctx);
    NOT_IN_SESSION(c);
    if (!img || !out || (flags & ~CRUM_VERIFY)) {
        set_detail("null image/out or bad flags");
        return CRUM_E_INVAL;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PreparedRestore pr;
    int st = prepare_restore(c, img->host, nullptr, img->len, s, flags, false, pr, false, true);
    if (st) {
        dev_free(pr.d_payload_tmp);
        return st;
    }
    auto *ss = new (std::nothrow) crum_restore_session;
    if (!ss) {
        dev_free(pr.d_payload_tmp);
        return CRUM_E_NOMEM;
    }
    ss->c = c;
    ss->img = img;
    ss->p = pr.p;
    ss->tab = pr.tab;
    ss->hst = pr.hst;
    ss->d_payload_tmp = pr.d_payload_tmp;
    ss->z_lazy = pr.z_lazy;
    ss->zsrc = pr.zsrc;

    const ParsedImage &p = ss->p;
    const uint64_t tail_len = p.image - p.ids_off;
    if ((st = dev_alloc(c, &ss->d_tail, tail_len + 16)) || (st = dev_alloc(c, &ss->d_rs, sizeof(RegStat) * (p.R + 1))) ||
        (st = dev_alloc(c, &ss->d_st, sizeof(DevStats))) || (st = dev_alloc(c, &ss->d_done, p.K + 1))) {
        session_free(ss);
        delete ss;
        return st;
    }
    if (ss->d_payload_tmp) {
        ss->payload_src = ss->d_payload_tmp;
    } else if (ss->z_lazy) {
        ss->payload_src = nullptr;  // windows decode into pool buffers
    } else {
        void *dp = nullptr;
        CK(cudaHostGetDevicePointer(&dp, img->host, 0));
        ss->payload_src = static_cast<const uint8_t *>(dp) + p.poff;
    }
    if (tail_len) CK(cudaMemcpyAsync(ss->d_tail, pr.d_ids, tail_len, cudaMemcpyDeviceToDevice, s));
    if (p.R) CK(cudaMemcpyAsync(ss->d_rs, c->d_rs, sizeof(RegStat) * p.R, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ss->d_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(ss->d_done, 0, p.K + 1, s));
    CK(cudaStreamSynchronize(s));
    ss->covered.assign(c->N, 0);
    ss->window.assign(p.R, 1);
    img->sessions++;
    c->session = ss;
    *out = ss;
    return CRUM_OK;
}

int crum_restore_fetch(crum_restore_session *ss, uint32_t region_id, uint64_t page, void *stream,
                       uint64_t *covered_out, uint64_t *restored_out) {
    if (!ss) {
        set_detail("null session");
        return CRUM_E_INVAL;
    }
    crum_ctx *c = ss->c;
    if (c->poisoned) {
        set_detail("context poisoned by an earlier CUDA error");
        return CRUM_E_CUDA;
    }
    CK(cudaSetDevice(c->device));
    uint32_t k = 0;
    while (k < c->regs.size() && c->regs[k].id != region_id) ++k;
    if (k == c->regs.size()) {
        set_detail("no region %u", region_id);
        return CRUM_E_NOREGION;
    }
    const HostRegion &h = c->regs[k];
    if (page >= h.n_pages) {
        set_detail("page %llu outside region %u", (unsigned long long)page, region_id);
        return CRUM_E_RANGE;
    }
    uint64_t newly = 0, restored = 0;
    uint8_t *cov = ss->covered.data() + h.page_base;
    if (!cov[page]) {
        // the window of this fault (sec. 4.2): whole small region; otherwise
        // `window` pages from the faulting one, clamped at the region end
        uint64_t lo = 0, hi = h.n_pages;
        if (h.n_pages > kSmallRegionPages) {
            lo = page;
            hi = page + std::min(ss->window[k], h.n_pages - page);
            if (ss->window[k] < (1ull << 62)) ss->window[k] *= 2;
        }
        const RegStat &r = ss->p.rs[k];
        const uint8_t *ids = ss->img->host + ss->p.ids_off;
        auto id_at = [&](uint64_t slot) { return (uint64_t)rd32(ids + 4 * slot); };
        // first slot of the region whose page id is >= x
        auto lower = [&](uint64_t x) {
            uint64_t a = r.first, b = r.first + r.n_dirty;
            while (a < b) {
                const uint64_t m = (a + b) / 2;
                if (id_at(m) < x) a = m + 1;
                else b = m;
            }
            return a;
        };
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        for (uint64_t x = lo; x < hi;) {
            if (cov[x]) {
                ++x;
                continue;
            }
            uint64_t y = x;
            while (y < hi && !cov[y]) cov[y++] = 1;
            newly += y - x;
            const uint64_t klo = lower(x), khi = lower(y);
            if (khi > klo) {
                int st = session_scatter_slots(ss, k, klo, khi, s);
                if (st) return st;
                restored += khi - klo;
            }
            x = y;
        }
        ss->covered_pages += newly;
        ss->restored += restored;
    }
    if (covered_out) *covered_out = newly;
    if (restored_out) *restored_out = restored;
    return CRUM_OK;
}

int crum_restore_end(crum_restore_session *ss, void *stream, crum_report *rep) {
    NvtxRange nvtx_("crum_restore_end");
    if (!ss) {
        set_detail("null session");
        return CRUM_E_INVAL;
    }
    crum_ctx *c = ss->c;
    int st = CRUM_OK;
    if (!c->poisoned && cudaSetDevice(c->device) == cudaSuccess) {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (ss->restored < ss->p.K && ss->z_lazy) {
            // compressed: the encoded payload crosses the link once, decodes in HBM
            const uint64_t units = ss->p.upayload >> kSegLog2;
            int e2 = grow(c, &c->d_renc, &c->renc_cap, ss->p.payload);
            if (!e2) e2 = grow(c, &c->d_rtmp, &c->rtmp_cap, ss->p.upayload);
            if (e2) {
                st = e2;
            } else {
                cudaMemcpyAsync(c->d_renc, ss->img->host + ss->p.poff, ss->p.payload, cudaMemcpyHostToDevice, s);
                const uint16_t *zsz = reinterpret_cast<const uint16_t *>(
                    ss->d_tail + tail_bytes_for(ss->p.K, (ss->p.flags & 2u) != 0));
                launch_zdecode(launch_of(c, s), c->d_renc, zsz, c->d_zloc, c->d_zblk, ss->d_st, c->d_rtmp, units, 0);
                ss->payload_src = c->d_rtmp;
            }
        }
        if (ss->restored < ss->p.K && st == CRUM_OK) {
            // every slot not yet written, in one launch (written ones skipped)
            ScatterArgs sa{};
            sa.regs = c->d_regs;
            sa.R = ss->p.R;
            sa.rs = ss->d_rs;
            sa.ids = reinterpret_cast<const uint32_t *>(ss->d_tail);
            sa.hashes = (ss->p.flags & 2u)
                            ? reinterpret_cast<const uint64_t *>(ss->d_tail + round_up(4 * ss->p.K, 8))
                            : nullptr;
            sa.st = ss->d_st;
            sa.src = ss->payload_src;
            sa.force = c->d_force;
            sa.u_lo = 0;
            sa.u_hi = ss->p.upayload >> kSegLog2;
            sa.skip = ss->d_done;
            launch_scatter(launch_of(c, s), sa);
        }
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_detail("lazy restore end: %s", cudaGetErrorString(e));
            c->poisoned = true;
            st = CRUM_E_CUDA;
        }
    } else {
        st = CRUM_E_CUDA;
    }
    if (rep) {
        memset(rep, 0, sizeof *rep);
        fill_report(c, ss->hst, rep);
        rep->image_bytes = ss->p.image;
    }
    session_free(ss);
    ss->img->sessions--;
    c->session = nullptr;
    delete ss;
    return st;
}

int crum_last_report(crum_ctx *ctx, crum_report *rep) {
    ENTER(ctx);
    if (!rep || c->last_kind == kLastNone) {
        set_detail(rep ? "no call to report on" : "null report");
        return CRUM_E_INVAL;
    }
    CK(cudaEventSynchronize(c->ev_done));
    CK(cudaMemcpy(c->h_st, c->d_st, sizeof(DevStats), cudaMemcpyDeviceToHost));
    memset(rep, 0, sizeof *rep);
    fill_report(c, *c->h_st, rep);
    if (c->last_timed) fill_times(c, *c->h_st, rep);
    else rep->path = (c->last_kind == kLastDevFused ? CRUM_PATH_FUSED : 0u) |
                     (c->last_kind == kLastDevFused && c->last_small ? CRUM_PATH_SMALL : 0u) | c->last_path;  // no times
    return CRUM_OK;
}

// ---------------------------------------------------------------------------
// test hooks
// ---------------------------------------------------------------------------
int crum_debug_detect(crum_ctx *ctx, void *stream, uint8_t *host_flags, uint64_t n) {
    ENTER(ctx);
    if (!host_flags || n != c->N) {
        set_detail("host_flags must hold exactly %llu pages", (unsigned long long)c->N);
        return CRUM_E_INVAL;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    enqueue_detect(c, s, c->all, false);
    launch_export_flags(launch_of(c, s), c->d_flags, c->d_force, c->N, kFlagTag, c->d_dbg);
    CK_LAUNCH();
    if (n) CK(cudaMemcpyAsync(host_flags, c->d_dbg, n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return CRUM_OK;
}

int crum_debug_export(crum_ctx *ctx, uint32_t id, int what, void *host_buf, uint64_t len) {
    ENTER(ctx);
    HostRegion *h = find_region(c, id);
    if (!h) return CRUM_E_NOREGION;
    if (!host_buf) return CRUM_E_INVAL;
    CK(cudaDeviceSynchronize());
    switch (what) {
        case CRUM_EXPORT_FORCE:
            if (len != h->n_pages) return CRUM_E_INVAL;
            CK(cudaMemcpy(host_buf, c->d_force + h->page_base, len, cudaMemcpyDeviceToHost));
            return CRUM_OK;
        case CRUM_EXPORT_HASHES:
            if (h->mode != kModeHash || len != 8 * h->n_pages) return CRUM_E_INVAL;
            CK(cudaMemcpy(host_buf, h->shadow, len, cudaMemcpyDeviceToHost));
            return CRUM_OK;
        case CRUM_EXPORT_MIRROR:
            if (h->mode != kModeCompare || len != h->bytes) return CRUM_E_INVAL;
            CK(cudaMemcpy(host_buf, h->shadow, len, cudaMemcpyDeviceToHost));
            return CRUM_OK;
        default:
            return CRUM_E_INVAL;
    }
}

}  // extern "C"
