/*
 * crum_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU model of CRUM's shadow-page
 * synchronisation (arXiv 1808.00117, Alg. 1 at PAPER.md:403-431, sec. 3.2 at
 * PAPER.md:433-444, sec. 3.4 drain/restart at PAPER.md:543-565), written to
 * the readings listed in DESIGN.md sec. "Readings".
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this code.  It shares no source, header,
 * table or constant with the CUDA path under paper_1808_00117_b200/.
 *
 * Everything is scalar C11: byte loops, memcmp/memcpy, a bit-at-a-time CRC-32
 * and XXH3-64 computed stripe by stripe in the library's documented order.
 * No blocking, fusion or reordering beyond what the definitions state.
 *
 * Pins (tests/test_oracle_*.py):
 *   orc_xxh3_64      -- python-xxhash xxh3_64_intdigest (library routine)
 *   orc_crc32        -- zlib.crc32 (library routine)
 *   orc_detect       -- brute-force Python bytes comparison, exhaustive flips
 *   sync / gather / restore -- invariants restore(ckpt(x)) == x, sync;sync==0,
 *                        dirty set == written set, numpy-assembled image bytes.
 *   lazy restore     -- fault count of a sequential read = ceil(log2(n+1)),
 *                        window sizes 1,2,4,..; windows hold the image's bytes
 *                        (independent parser) and nothing else changes;
 *                        begin+fetches+end == restore_scatter.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status codes: the values are the ABI contract of include/crum.h (restated
 * here, not included, so the oracle stays independent of the product). */
enum {
    ORC_OK = 0,
    ORC_E_INVAL = -1,
    ORC_E_OVERLAP = -2,
    ORC_E_NOREGION = -3,
    ORC_E_RANGE = -4,
    ORC_E_NOMEM = -5,
    ORC_E_CAPACITY = -6,
    ORC_E_CORRUPT = -7,
    ORC_E_MISMATCH = -8,
    ORC_E_BUSY = -9,
};

enum { ORC_MODE_COMPARE = 0, ORC_MODE_HASH = 1, ORC_MODE_TRACKED = 2 };
enum { ORC_FULL = 1u, ORC_VERIFY = 2u, ORC_COMPRESS = 4u };
enum { ORC_IMG_FULL = 1u, ORC_IMG_HAS_HASHES = 2u, ORC_IMG_COMPRESSED = 4u };

#define ORC_MIN_PAGE 4096ull
#define ORC_MAX_PAGE (2ull << 20)
#define ORC_MAX_TOTAL_PAGES 0x7fffffffull

typedef struct {
    uint64_t scanned_pages, scanned_bytes;
    uint64_t dirty_pages, dirty_bytes, dirty_runs;
    uint64_t image_bytes;
} orc_report;

typedef struct {
    uint32_t id;
    uint32_t mode;
    uint8_t *cur;        /* the registered bytes ("real" pages, Q5) */
    uint64_t bytes;      /* B_r */
    uint64_t page_size;  /* P_r */
    uint64_t n_pages;    /* n_r = ceil(B_r / P_r) */
    uint8_t *mirror;     /* compare mode: last committed bytes (B_r) */
    uint64_t *table;     /* hash mode: last committed XXH3 per page */
    uint8_t *force;      /* per-page force-dirty bit (Q3) */
} orc_region;

/* An open lazy restore (sec. 4.2 read-fault heuristic applied to restart). */
typedef struct {
    const uint8_t *img;  /* the validated image (caller keeps it alive) */
    uint8_t *upay;       /* decoded payload of a compressed image (owned), or NULL */
    uint8_t **present;   /* per region, per page: read in already */
    uint64_t *window;    /* per region: pages the next fault reads */
    uint8_t *written;    /* per slot: restored already */
} orc_session;

typedef struct {
    orc_region *r;       /* ascending id order */
    uint32_t n;
    uint32_t next_id;
    orc_session *sess;   /* open lazy restore, or NULL */
} orc_ctx;

/* ------------------------------------------------------------------ */
/* Little-endian helpers (byte by byte, host-endianness independent).  */
/* ------------------------------------------------------------------ */
static uint64_t rd64(const uint8_t *p)
{
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}
static uint32_t rd32(const uint8_t *p)
{
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
static void wr64(uint8_t *p, uint64_t v)
{
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static void wr32(uint8_t *p, uint32_t v)
{
    for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

/* ------------------------------------------------------------------ */
/* CRC-32 (zlib polynomial, reflected 0xEDB88320, init/final ~0),      */
/* one bit at a time -- the textbook definition.                       */
/* ------------------------------------------------------------------ */
uint32_t orc_crc32(const uint8_t *p, uint64_t n)
{
    uint32_t c = 0xffffffffu;
    for (uint64_t i = 0; i < n; ++i) {
        c ^= p[i];
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xedb88320u & (0u - (c & 1u)));
    }
    return c ^ 0xffffffffu;
}

/* ------------------------------------------------------------------ */
/* XXH3-64, seed 0, default secret, long-input path (len > 240).       */
/* Reading Q8: the per-page hash is XXH3_64bits of the     */
/* zero-padded P-byte slot.  Steps follow xxhash 0.8's documented long */
/* loop: stripes of 64 B, blocks of 16 stripes, scramble after each    */
/* full block, a partial last block, the last stripe at secret offset  */
/* 121, merge at secret offset 11, avalanche.                          */
/* ------------------------------------------------------------------ */
static const uint8_t orc_secret[192] = {
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

#define ORC_P32_1 0x9E3779B1ull
#define ORC_P32_2 0x85EBCA77ull
#define ORC_P32_3 0xC2B2AE3Dull
#define ORC_P64_1 0x9E3779B185EBCA87ull
#define ORC_P64_2 0xC2B2AE3D27D4EB4Full
#define ORC_P64_3 0x165667B19E3779F9ull
#define ORC_P64_4 0x85EBCA77C2B2AE63ull
#define ORC_P64_5 0x27D4EB2F165667C5ull
#define ORC_PMX1 0x165667919E3779F9ull

/* One 64-byte stripe into the 8 accumulators, secret at byte offset `so`. */
static void orc_accumulate_stripe(uint64_t acc[8], const uint8_t *in, uint64_t so)
{
    for (int l = 0; l < 8; ++l) {
        uint64_t v = rd64(in + 8 * l);
        uint64_t k = v ^ rd64(orc_secret + so + 8 * l);
        acc[l ^ 1] += v;
        acc[l] += (k & 0xffffffffull) * (k >> 32);
    }
}

static void orc_scramble(uint64_t acc[8])
{
    for (int l = 0; l < 8; ++l) {
        uint64_t a = acc[l];
        a ^= a >> 47;
        a ^= rd64(orc_secret + 128 + 8 * l);
        a *= ORC_P32_1;
        acc[l] = a;
    }
}

/* 64x64 -> 128 multiply folded (lo ^ hi), from 32-bit halves. */
static uint64_t orc_mul128_fold64(uint64_t a, uint64_t b)
{
    uint64_t a0 = a & 0xffffffffull, a1 = a >> 32;
    uint64_t b0 = b & 0xffffffffull, b1 = b >> 32;
    uint64_t p00 = a0 * b0, p01 = a0 * b1, p10 = a1 * b0, p11 = a1 * b1;
    uint64_t mid = (p00 >> 32) + (p10 & 0xffffffffull) + p01;
    uint64_t lo = (mid << 32) | (p00 & 0xffffffffull);
    uint64_t hi = p11 + (p10 >> 32) + (mid >> 32);
    return lo ^ hi;
}

/* Returns 0 for len <= 240 (outside the oracle's contract; all slots are
 * >= 4096 bytes). */
uint64_t orc_xxh3_64(const uint8_t *in, uint64_t len)
{
    if (len <= 240) return 0;
    uint64_t acc[8] = {ORC_P32_3, ORC_P64_1, ORC_P64_2, ORC_P64_3,
                       ORC_P64_4, ORC_P32_2, ORC_P64_5, ORC_P32_1};
    const uint64_t stripes_per_block = (192 - 64) / 8; /* 16 */
    const uint64_t block_len = 64 * stripes_per_block; /* 1024 */
    const uint64_t nb = (len - 1) / block_len;
    for (uint64_t b = 0; b < nb; ++b) {
        for (uint64_t s = 0; s < stripes_per_block; ++s)
            orc_accumulate_stripe(acc, in + b * block_len + 64 * s, 8 * s);
        orc_scramble(acc);
    }
    const uint64_t last_stripes = ((len - 1) - block_len * nb) / 64;
    for (uint64_t s = 0; s < last_stripes; ++s)
        orc_accumulate_stripe(acc, in + nb * block_len + 64 * s, 8 * s);
    orc_accumulate_stripe(acc, in + len - 64, 192 - 64 - 7);
    uint64_t r = len * ORC_P64_1;
    for (int i = 0; i < 4; ++i)
        r += orc_mul128_fold64(acc[2 * i] ^ rd64(orc_secret + 11 + 16 * i),
                               acc[2 * i + 1] ^ rd64(orc_secret + 11 + 16 * i + 8));
    r ^= r >> 37;
    r *= ORC_PMX1;
    r ^= r >> 32;
    return r;
}

/* ------------------------------------------------------------------ */
/* Region bookkeeping.                                                 */
/* ------------------------------------------------------------------ */
static uint64_t page_len(const orc_region *g, uint64_t i)
{
    uint64_t off = i * g->page_size;
    uint64_t rest = g->bytes - off;
    return rest < g->page_size ? rest : g->page_size;
}

/* H(r,i): XXH3 of the page's logical bytes followed by zero padding to P. */
static uint64_t page_hash(const orc_region *g, uint64_t i)
{
    uint64_t len = page_len(g, i);
    if (len == g->page_size) return orc_xxh3_64(g->cur + i * g->page_size, len);
    uint8_t *slot = (uint8_t *)calloc(1, g->page_size);
    memcpy(slot, g->cur + i * g->page_size, len);
    uint64_t h = orc_xxh3_64(slot, g->page_size);
    free(slot);
    return h;
}

static orc_region *find(orc_ctx *c, uint32_t id)
{
    for (uint32_t k = 0; k < c->n; ++k)
        if (c->r[k].id == id) return &c->r[k];
    return NULL;
}

static uint64_t total_pages(const orc_ctx *c)
{
    uint64_t n = 0;
    for (uint32_t k = 0; k < c->n; ++k) n += c->r[k].n_pages;
    return n;
}

orc_ctx *orc_create(void)
{
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    if (c) c->next_id = 1;
    return c;
}

static void free_region(orc_region *g)
{
    free(g->mirror);
    free(g->table);
    free(g->force);
}

void orc_destroy(orc_ctx *c)
{
    if (!c) return;
    if (c->sess) {
        for (uint32_t k = 0; k < c->n; ++k) free(c->sess->present[k]);
        free(c->sess->present);
        free(c->sess->window);
        free(c->sess->written);
        free(c->sess->upay);
        free(c->sess);
    }
    for (uint32_t k = 0; k < c->n; ++k) free_region(&c->r[k]);
    free(c->r);
    free(c);
}

/* Alg. 1 "CUDA Create UVM region" + "all the pages in
 * the regions are marked as dirty": force[] = 1. */
int orc_register_region(orc_ctx *c, uint8_t *ptr, uint64_t bytes, uint64_t page_size,
                        uint32_t mode, uint32_t *id_out)
{
    if (c && c->sess) return ORC_E_BUSY;
    if (!c || !ptr || !id_out || bytes == 0) return ORC_E_INVAL;
    if (page_size < ORC_MIN_PAGE || page_size > ORC_MAX_PAGE || (page_size & (page_size - 1)))
        return ORC_E_INVAL;
    if (((uintptr_t)ptr) % 16 != 0) return ORC_E_INVAL;
    if (mode != ORC_MODE_COMPARE && mode != ORC_MODE_HASH && mode != ORC_MODE_TRACKED) return ORC_E_INVAL;
    uint64_t n = bytes / page_size + (bytes % page_size != 0);
    if (n > 0xffffffffull) return ORC_E_INVAL;
    if (total_pages(c) + n > ORC_MAX_TOTAL_PAGES) return ORC_E_INVAL;
    uintptr_t lo = (uintptr_t)ptr, hi = lo + bytes;
    for (uint32_t k = 0; k < c->n; ++k) {
        uintptr_t a = (uintptr_t)c->r[k].cur, b = a + c->r[k].bytes;
        if (lo < b && a < hi) return ORC_E_OVERLAP;
    }
    orc_region g;
    memset(&g, 0, sizeof g);
    g.mode = mode;
    g.cur = ptr;
    g.bytes = bytes;
    g.page_size = page_size;
    g.n_pages = n;
    g.force = (uint8_t *)malloc(n);
    if (mode == ORC_MODE_COMPARE) g.mirror = (uint8_t *)calloc(1, bytes);
    else if (mode == ORC_MODE_HASH) g.table = (uint64_t *)calloc(n, sizeof(uint64_t));
    orc_region *nr = (orc_region *)realloc(c->r, (c->n + 1) * sizeof(orc_region));
    if (!g.force || (mode != ORC_MODE_TRACKED && !g.mirror && !g.table) || !nr) {
        free_region(&g);
        if (nr) c->r = nr;
        return ORC_E_NOMEM;
    }
    c->r = nr;
    memset(g.force, 1, n);
    g.id = c->next_id++;
    c->r[c->n++] = g;
    *id_out = g.id;
    return ORC_OK;
}

int orc_unregister_region(orc_ctx *c, uint32_t id)
{
    if (c && c->sess) return ORC_E_BUSY;
    if (!c) return ORC_E_INVAL;
    for (uint32_t k = 0; k < c->n; ++k) {
        if (c->r[k].id != id) continue;
        free_region(&c->r[k]);
        memmove(&c->r[k], &c->r[k + 1], (c->n - k - 1) * sizeof(orc_region));
        c->n--;
        return ORC_OK;
    }
    return ORC_E_NOREGION;
}

/* MarkPageAsDirty (Alg. 1) as an explicit call: every page
 * overlapping [off, off+len) gets its force bit. */
int orc_mark_dirty(orc_ctx *c, uint32_t id, uint64_t off, uint64_t len)
{
    if (!c) return ORC_E_INVAL;
    orc_region *g = find(c, id);
    if (!g) return ORC_E_NOREGION;
    if (off > g->bytes || len > g->bytes - off) return ORC_E_RANGE;
    if (len == 0) return ORC_OK;
    for (uint64_t i = off / g->page_size; i <= (off + len - 1) / g->page_size; ++i) g->force[i] = 1;
    return ORC_OK;
}

/* Batch form of MarkPageAsDirty: force bits of the listed page indices. */
int orc_mark_pages(orc_ctx *c, uint32_t id, const uint32_t *pages, uint64_t n)
{
    if (!c || (!pages && n)) return ORC_E_INVAL;
    orc_region *g = find(c, id);
    if (!g) return ORC_E_NOREGION;
    for (uint64_t k = 0; k < n; ++k)
        if (pages[k] >= g->n_pages) return ORC_E_RANGE;
    for (uint64_t k = 0; k < n; ++k) g->force[pages[k]] = 1;
    return ORC_OK;
}

/* Detect (pure): D_r = { i : force[i] or content changed since commit }.
 * Reading Q1: "dirty" = bytes differ from the last committed snapshot
 * (compare: memcmp over the logical length; hash: H(r,i) != table[i]).
 * TRACKED mode is the paper's own write-based rule (Alg. 1 MarkPageAsDirty,
 * PAPER.md:412): a page is dirty iff it was marked since its last commit. */
static int page_dirty(const orc_region *g, uint64_t i)
{
    if (g->force[i]) return 1;
    if (g->mode == ORC_MODE_TRACKED) return 0;
    if (g->mode == ORC_MODE_COMPARE) {
        uint64_t off = i * g->page_size;
        return memcmp(g->cur + off, g->mirror + off, page_len(g, i)) != 0;
    }
    return page_hash(g, i) != g->table[i];
}

int orc_detect(orc_ctx *c, uint32_t id, uint8_t *flags_out)
{
    if (!c || !flags_out) return ORC_E_INVAL;
    orc_region *g = find(c, id);
    if (!g) return ORC_E_NOREGION;
    for (uint64_t i = 0; i < g->n_pages; ++i) flags_out[i] = (uint8_t)page_dirty(g, i);
    return ORC_OK;
}

/* Commit (ClearDirtyPages): snapshot <- current, force <- 0. */
static void commit_page(orc_region *g, uint64_t i)
{
    if (g->mode == ORC_MODE_COMPARE) {
        uint64_t off = i * g->page_size;
        memcpy(g->mirror + off, g->cur + off, page_len(g, i));
    } else if (g->mode == ORC_MODE_HASH) {
        g->table[i] = page_hash(g, i);
    }
    g->force[i] = 0;
}

/* Alg. 1 "CUDA call": for r ascending, detect D_r and
 * commit all of it; return sum |D_r|. */
int orc_sync_shadow(orc_ctx *c, uint64_t *n_out)
{
    if (c && c->sess) return ORC_E_BUSY;
    if (!c) return ORC_E_INVAL;
    uint64_t total = 0;
    for (uint32_t k = 0; k < c->n; ++k) {
        orc_region *g = &c->r[k];
        for (uint64_t i = 0; i < g->n_pages; ++i) {
            if (page_dirty(g, i)) {
                commit_page(g, i);
                total++;
            }
        }
    }
    if (n_out) *n_out = total;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Image format v1 (reading Q10).            */
/* ------------------------------------------------------------------ */
static uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

/* Layout: header | table | zero pad | payload | ids | hashes. */
static uint64_t payload_offset_for(uint64_t R) { return round_up(64 + 48 * R, 4096); }

static uint64_t tail_bytes_for(uint64_t K, int has_hashes)
{
    return round_up(4 * K, 8) + (has_hashes ? 8 * K : 0);
}

/* zlib CRC-32 of the concatenation a || b (one bit at a time). */
static uint32_t crc32_two(const uint8_t *a, uint64_t na, const uint8_t *b, uint64_t nb)
{
    uint32_t c = 0xffffffffu;
    for (uint64_t i = 0; i < na + nb; ++i) {
        c ^= i < na ? a[i] : b[i - na];
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xedb88320u & (0u - (c & 1u)));
    }
    return c ^ 0xffffffffu;
}

static int any_hash_region(const orc_ctx *c)
{
    for (uint32_t k = 0; k < c->n; ++k)
        if (c->r[k].mode == ORC_MODE_HASH) return 1;
    return 0;
}

/* Worst-case image size when at most max_dirty pages are listed. */
int orc_image_required_bytes(orc_ctx *c, uint64_t max_dirty, uint64_t *out)
{
    if (!c || !out) return ORC_E_INVAL;
    uint64_t N = total_pages(c), K = max_dirty < N ? max_dirty : N;
    uint64_t payload = 0, maxp = 0;
    for (uint32_t k = 0; k < c->n; ++k) {
        payload += c->r[k].n_pages * c->r[k].page_size;
        if (c->r[k].page_size > maxp) maxp = c->r[k].page_size;
    }
    if (K < N && K * maxp < payload) payload = K * maxp;
    /* + the unit-size table a compressed image carries (reading Z2) */
    *out = payload_offset_for(c->n) + payload + tail_bytes_for(K, any_hash_region(c)) +
           round_up(2 * (payload / 4096), 8);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Unit codec of compressed images (readings  */
/* Z2-Z3 in DESIGN.md).  The paper compresses the image with gzip -1  */
/* or LZ4 before writing it (Table 2): an LZ77      */
/* match finder plus an entropy coder.  Here every 4096-byte unit is  */
/* encoded on its own (reading Z3):                                   */
/*   all bytes zero          -> nothing (encoded size 0)              */
/*   else the DEFLATE stream below if it is shorter than 4096 bytes,  */
/*   else the 4096 raw bytes (encoded size 4096).                     */
/* The DEFLATE stream (RFC 1951) is ONE block, BFINAL = 1, BTYPE = 01 */
/* (the fixed Huffman codes of RFC 1951 sec. 3.2.6), zero-padded to a */
/* whole byte, holding this greedy LZ77 parse of the unit u[0..4096): */
/*   h(p)    = ((LE u32 at u+p) * 2654435761 mod 2^32) >> 20,         */
/*             for p <= 4092 (a 12-bit hash of the 4 bytes at p);    */
/*   cand(p) = the largest q < p with h(q) == h(p) -- every position */
/*             enters the hash table, whether the parse stops there  */
/*             or not;                                               */
/*   len(p)  = the largest L <= min(258, 4096 - p) with               */
/*             u[cand(p) + i] == u[p + i] for all i < L (0 if no      */
/*             cand; the copy may overlap p);                        */
/*   parse:  p = 0; while p < 4096: if len(p) >= 4 emit the match     */
/*           (len(p), distance p - cand(p)) and p += len(p), else     */
/*           emit the literal u[p] and p += 1; then end-of-block.     */
/* ------------------------------------------------------------------ */
#define ORC_UNIT 4096ull
#define Z_HASH_BITS 12
#define Z_MAX_MATCH 258u
#define Z_MIN_MATCH 4u

/* RFC 1951 sec. 3.2.5: length codes 257..285 (base length, extra bits) and
 * distance codes 0..29 (base distance, extra bits), written out as tables. */
static const uint16_t z_len_base[29] = {3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31,
                                        35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
static const uint8_t z_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2,
                                        3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
static const uint16_t z_dist_base[30] = {1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193,
                                         257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145,
                                         8193, 12289, 16385, 24577};
static const uint8_t z_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6,
                                         7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

/* Bit writer: bits go LSB-first into bytes (RFC 1951 sec. 3.1.1). */
typedef struct {
    uint8_t *out;
    uint64_t cap, nbits;
} z_bits;

static void z_put(z_bits *w, uint32_t v, uint32_t n) /* n low bits of v, LSB first */
{
    for (uint32_t i = 0; i < n; ++i, ++w->nbits) {
        const uint64_t byte = w->nbits / 8;
        if (byte >= w->cap) continue; /* counted, not stored: the caller falls back to raw */
        if ((v >> i) & 1u) w->out[byte] |= (uint8_t)(1u << (w->nbits % 8));
    }
}

/* A Huffman code is packed starting with its most significant bit. */
static void z_put_code(z_bits *w, uint32_t code, uint32_t n)
{
    for (uint32_t i = 0; i < n; ++i) z_put(w, (code >> (n - 1 - i)) & 1u, 1);
}

/* Fixed literal/length code of symbol s (RFC 1951 sec. 3.2.6). */
static void z_put_litlen(z_bits *w, uint32_t s)
{
    if (s <= 143) z_put_code(w, 0x30 + s, 8);
    else if (s <= 255) z_put_code(w, 0x190 + (s - 144), 9);
    else if (s <= 279) z_put_code(w, s - 256, 7);
    else z_put_code(w, 0xC0 + (s - 280), 8);
}

static void z_put_match(z_bits *w, uint32_t len, uint32_t dist)
{
    uint32_t lc = 28;
    while (z_len_base[lc] > len) --lc;       /* largest base <= len (258 -> code 285) */
    z_put_litlen(w, 257 + lc);
    z_put(w, len - z_len_base[lc], z_len_extra[lc]);
    uint32_t dc = 29;
    while (z_dist_base[dc] > dist) --dc;
    z_put_code(w, dc, 5);                     /* fixed distance codes: 5 bits */
    z_put(w, dist - z_dist_base[dc], z_dist_extra[dc]);
}

static uint32_t z_hash(const uint8_t *u, uint64_t p)
{
    return (uint32_t)(rd32(u + p) * 2654435761u) >> (32 - Z_HASH_BITS);
}

/* Encode one unit into out (room for 4096 bytes); returns the encoded size. */
uint64_t orc_z_encode(const uint8_t *u, uint8_t *out)
{
    int zero = 1;
    for (uint64_t i = 0; i < ORC_UNIT; ++i) zero &= u[i] == 0;
    if (zero) return 0;
    /* cand(p) for every p: the hash table sees every position in order */
    int32_t head[1 << Z_HASH_BITS];
    int32_t cand[ORC_UNIT];
    for (uint32_t h = 0; h < (1u << Z_HASH_BITS); ++h) head[h] = -1;
    for (uint64_t p = 0; p < ORC_UNIT; ++p) {
        cand[p] = -1;
        if (p + 4 <= ORC_UNIT) {
            const uint32_t h = z_hash(u, p);
            cand[p] = head[h];
            head[h] = (int32_t)p;
        }
    }
    memset(out, 0, ORC_UNIT);
    z_bits w = {out, ORC_UNIT, 0};
    z_put(&w, 1, 1); /* BFINAL */
    z_put(&w, 1, 2); /* BTYPE = 01: fixed Huffman codes */
    uint64_t p = 0;
    while (p < ORC_UNIT) {
        uint32_t len = 0;
        if (cand[p] >= 0) {
            const uint64_t q = (uint64_t)cand[p];
            const uint64_t lim = ORC_UNIT - p < Z_MAX_MATCH ? ORC_UNIT - p : Z_MAX_MATCH;
            while (len < lim && u[q + len] == u[p + len]) ++len;
        }
        if (len >= Z_MIN_MATCH) {
            z_put_match(&w, len, (uint32_t)(p - (uint64_t)cand[p]));
            p += len;
        } else {
            z_put_litlen(&w, u[p]);
            p += 1;
        }
    }
    z_put_litlen(&w, 256); /* end of block */
    const uint64_t nbytes = (w.nbits + 7) / 8;
    if (nbytes >= ORC_UNIT) {
        memcpy(out, u, ORC_UNIT);
        return ORC_UNIT;
    }
    return nbytes;
}

/* A valid encoded size: anything up to 4096 (what the bytes hold is checked
 * by the decoder). */
static int z_size_ok(uint64_t cs) { return cs <= ORC_UNIT; }

/* Bit reader over the cs bytes of a stream. */
typedef struct {
    const uint8_t *in;
    uint64_t nbits, pos;
    int overrun;
} z_in;

static uint32_t z_get(z_in *r, uint32_t n) /* n bits, LSB first */
{
    uint32_t v = 0;
    for (uint32_t i = 0; i < n; ++i, ++r->pos) {
        if (r->pos >= r->nbits) {
            r->overrun = 1;
            continue;
        }
        v |= (uint32_t)((r->in[r->pos / 8] >> (r->pos % 8)) & 1u) << i;
    }
    return v;
}

/* Next fixed literal/length symbol, or -1 (RFC 1951 sec. 3.2.6: codes 286,
 * 287 do not occur in a valid stream). */
static int z_get_litlen(z_in *r)
{
    uint32_t c = 0;
    for (uint32_t n = 1; n <= 9; ++n) {
        c = (c << 1) | z_get(r, 1);
        if (n == 7 && c <= 0x17) return (int)(256 + c);
        if (n == 8 && c >= 0x30 && c <= 0xBF) return (int)(c - 0x30);
        if (n == 8 && c >= 0xC0 && c <= 0xC5) return (int)(280 + c - 0xC0);
        if (n == 8 && c >= 0xC6 && c <= 0xC7) return -1;
        if (n == 9 && c >= 0x190) return (int)(144 + c - 0x190);
    }
    return -1;
}

/* Decode one unit of encoded size cs from in; 0 if the bytes are not a valid
 * encoding: a size-0 unit is zero, a size-4096 unit is raw; otherwise the
 * bytes must be exactly one final fixed-Huffman block that produces exactly
 * 4096 bytes, every distance within the bytes already produced, ending in
 * the last byte with zero padding bits. */
int orc_z_decode(const uint8_t *in, uint64_t cs, uint8_t *u)
{
    if (!z_size_ok(cs)) return 0;
    if (cs == ORC_UNIT) {
        memcpy(u, in, ORC_UNIT);
        return 1;
    }
    memset(u, 0, ORC_UNIT);
    if (cs == 0) return 1;
    z_in r = {in, 8 * cs, 0, 0};
    if (z_get(&r, 1) != 1 || z_get(&r, 2) != 1) return 0; /* BFINAL = 1, BTYPE = 01 */
    uint64_t o = 0;
    for (;;) {
        const int s = z_get_litlen(&r);
        if (s < 0 || r.overrun) return 0;
        if (s == 256) break;
        if (s < 256) {
            if (o >= ORC_UNIT) return 0;
            u[o++] = (uint8_t)s;
            continue;
        }
        const uint32_t lc = (uint32_t)s - 257;
        const uint32_t len = z_len_base[lc] + z_get(&r, z_len_extra[lc]);
        uint32_t dc = 0;
        for (int i = 0; i < 5; ++i) dc = (dc << 1) | z_get(&r, 1);
        if (dc >= 30 || r.overrun) return 0;
        const uint32_t dist = z_dist_base[dc] + z_get(&r, z_dist_extra[dc]);
        if (r.overrun || dist > o || o + len > ORC_UNIT) return 0;
        for (uint32_t i = 0; i < len; ++i, ++o) u[o] = u[o - dist];
    }
    if (o != ORC_UNIT) return 0;
    /* the stream ends in its last byte and the padding bits are zero */
    if ((r.pos + 7) / 8 != cs) return 0;
    while (r.pos < r.nbits)
        if (z_get(&r, 1)) return 0;
    return 1;
}

/* Checkpoint drain as an incremental gather (sec. 3.4, PAPER.md:547-551;
 * readings Q5, Q12): list D_r (or every page under FULL) for r ascending,
 * assemble the v1 image, then commit every listed page.  On CAPACITY nothing
 * changes and report->image_bytes holds the required size. */
int orc_checkpoint_gather(orc_ctx *c, uint32_t flags, uint8_t *img, uint64_t cap,
                          orc_report *rep)
{
    if (c && c->sess) return ORC_E_BUSY;
    if (!c || !img || (flags & ~(ORC_FULL | ORC_COMPRESS))) return ORC_E_INVAL;
    const uint32_t R = c->n;
    uint64_t N = total_pages(c);
    /* Step 1: the listed pages (global order: region table order, page index). */
    uint8_t **listed = (uint8_t **)calloc(R ? R : 1, sizeof(uint8_t *));
    uint64_t K = 0, payload = 0, dirty_bytes = 0, runs = 0, scanned_bytes = 0;
    for (uint32_t k = 0; k < R; ++k) {
        orc_region *g = &c->r[k];
        listed[k] = (uint8_t *)calloc(g->n_pages, 1);
        scanned_bytes += g->bytes;
        for (uint64_t i = 0; i < g->n_pages; ++i) {
            listed[k][i] = (flags & ORC_FULL) ? 1 : (uint8_t)page_dirty(g, i);
            if (!listed[k][i]) continue;
            K++;
            payload += g->page_size;
            dirty_bytes += page_len(g, i);
            if (i == 0 || !listed[k][i - 1]) runs++;
        }
    }
    const int has_hashes = any_hash_region(c);
    const int z = (flags & ORC_COMPRESS) != 0;
    const uint64_t poff = payload_offset_for(R);
    /* Compressed images (readings Z2-Z3): the slots are laid out as usual,
     * then every 4 KiB unit is encoded; the payload is the encoded units back
     * to back, zero-padded to a multiple of 4096; the tail gains the u16
     * encoded size of every unit. */
    const uint64_t U = payload / ORC_UNIT;
    uint8_t *zbuf = NULL;
    uint16_t *zsz = NULL;
    uint64_t zbytes = 0;
    if (z) {
        uint8_t *upay = (uint8_t *)calloc(payload ? payload : 1, 1);
        uint64_t pb = 0;
        for (uint32_t k = 0; k < R; ++k) {
            orc_region *g = &c->r[k];
            for (uint64_t i = 0; i < g->n_pages; ++i) {
                if (!listed[k][i]) continue;
                memcpy(upay + pb, g->cur + i * g->page_size, page_len(g, i));
                pb += g->page_size;
            }
        }
        zbuf = (uint8_t *)malloc(payload ? payload : 1);
        zsz = (uint16_t *)malloc(U ? 2 * U : 2);
        for (uint64_t u = 0; u < U; ++u) {
            uint64_t cs = orc_z_encode(upay + u * ORC_UNIT, zbuf + zbytes);
            zsz[u] = (uint16_t)(cs == ORC_UNIT ? 4096 : cs);
            zbytes += cs;
        }
        free(upay);
    }
    const uint64_t pay_field = z ? round_up(zbytes, ORC_UNIT) : payload;
    const uint64_t ids_off = poff + pay_field;
    const uint64_t total = ids_off + tail_bytes_for(K, has_hashes) + (z ? round_up(2 * U, 8) : 0);
    if (rep) {
        rep->scanned_pages = N;
        rep->scanned_bytes = scanned_bytes;
        rep->dirty_pages = K;
        rep->dirty_bytes = dirty_bytes;
        rep->dirty_runs = runs;
        rep->image_bytes = total;
    }
    if (cap < total) {
        for (uint32_t k = 0; k < R; ++k) free(listed[k]);
        free(listed);
        free(zbuf);
        free(zsz);
        return ORC_E_CAPACITY;
    }
    /* Step 2: assemble. */
    memset(img, 0, total);
    memcpy(img, "CRUM", 4);
    wr32(img + 4, 1);
    wr32(img + 8, ((flags & ORC_FULL) ? ORC_IMG_FULL : 0) | (has_hashes ? ORC_IMG_HAS_HASHES : 0) |
                      (z ? ORC_IMG_COMPRESSED : 0));
    wr32(img + 12, R);
    wr64(img + 16, K);
    wr64(img + 24, poff);
    wr64(img + 32, pay_field);
    wr64(img + 40, ids_off);
    wr64(img + 48, total);
    uint8_t *tab = img + 64;
    uint8_t *ids = img + ids_off;
    uint8_t *hashes = ids + round_up(4 * K, 8);
    uint64_t slot = 0, pbyte = 0;
    for (uint32_t k = 0; k < R; ++k) {
        orc_region *g = &c->r[k];
        uint64_t nd = 0, first = slot;
        for (uint64_t i = 0; i < g->n_pages; ++i) {
            if (!listed[k][i]) continue;
            wr32(ids + 4 * slot, (uint32_t)i);
            if (has_hashes) wr64(hashes + 8 * slot, g->mode == ORC_MODE_HASH ? page_hash(g, i) : 0);
            if (!z) memcpy(img + poff + pbyte, g->cur + i * g->page_size, page_len(g, i));
            pbyte += g->page_size;
            slot++;
            nd++;
        }
        uint8_t *e = tab + 48 * (uint64_t)k;
        wr32(e + 0, g->id);
        wr32(e + 4, g->mode);
        wr64(e + 8, g->bytes);
        wr64(e + 16, g->page_size);
        wr64(e + 24, g->n_pages);
        wr64(e + 32, nd);
        wr64(e + 40, first);
    }
    if (z) {
        memcpy(img + poff, zbuf, zbytes);
        uint8_t *zt = ids + tail_bytes_for(K, has_hashes);
        for (uint64_t u = 0; u < U; ++u) {
            zt[2 * u] = (uint8_t)zsz[u];
            zt[2 * u + 1] = (uint8_t)(zsz[u] >> 8);
        }
        free(zbuf);
        free(zsz);
    }
    wr32(img + 56, crc32_two(tab, 48 * (uint64_t)R, ids, total - ids_off));
    wr32(img + 60, orc_crc32(img, 60));
    /* Step 3: commit every listed page. */
    for (uint32_t k = 0; k < R; ++k) {
        for (uint64_t i = 0; i < c->r[k].n_pages; ++i)
            if (listed[k][i]) commit_page(&c->r[k], i);
        free(listed[k]);
    }
    free(listed);
    return ORC_OK;
}

/* Every check a restore makes before writing anything (reading Q11). */
/* *upay_out: for a compressed image, the decoded payload (malloc'ed, the
 * caller frees it); NULL otherwise (the payload is read in place). */
static int validate_image(orc_ctx *c, const uint8_t *img, uint64_t len, uint32_t flags, uint8_t **upay_out)
{
    *upay_out = NULL;
    if (len < 64 || memcmp(img, "CRUM", 4) != 0) return ORC_E_CORRUPT;
    if (orc_crc32(img, 60) != rd32(img + 60)) return ORC_E_CORRUPT;
    const uint32_t version = rd32(img + 4), iflags = rd32(img + 8), R = rd32(img + 12);
    const uint64_t K = rd64(img + 16), poff = rd64(img + 24), payload = rd64(img + 32),
                   ids_off = rd64(img + 40), total = rd64(img + 48);
    if (version != 1 || (iflags & ~7u) != 0) return ORC_E_CORRUPT;
    const int has_hashes = (iflags & ORC_IMG_HAS_HASHES) != 0;
    const int z = (iflags & ORC_IMG_COMPRESSED) != 0;
    if (K > ORC_MAX_TOTAL_PAGES || R > 0x7fffffffu) return ORC_E_CORRUPT;
    if (poff != payload_offset_for(R) || payload > (1ull << 62) || ids_off != poff + payload)
        return ORC_E_CORRUPT;
    if (!z && total != ids_off + tail_bytes_for(K, has_hashes)) return ORC_E_CORRUPT;
    /* compressed: the exact length needs the unit count (from the table) */
    if (z && (payload % ORC_UNIT != 0 || total < ids_off + tail_bytes_for(K, has_hashes) ||
              total > ids_off + tail_bytes_for(K, has_hashes) + (1ull << 62)))
        return ORC_E_CORRUPT;
    if (len < total) return ORC_E_CORRUPT;
    const uint8_t *tab = img + 64;
    const uint8_t *ids = img + ids_off;
    const uint8_t *hashes = ids + round_up(4 * K, 8);
    if (crc32_two(tab, 48 * (uint64_t)R, ids, total - ids_off) != rd32(img + 56)) return ORC_E_CORRUPT;
    /* Structural consistency of the table, ids and hash list. */
    uint64_t sum = 0, pay = 0;
    int any_hash = 0;
    for (uint32_t k = 0; k < R; ++k) {
        const uint8_t *e = tab + 48 * (uint64_t)k;
        uint32_t mode = rd32(e + 4);
        uint64_t bytes = rd64(e + 8), ps = rd64(e + 16), np = rd64(e + 24), nd = rd64(e + 32),
                 first = rd64(e + 40);
        if (mode > 2 || ps < ORC_MIN_PAGE || ps > ORC_MAX_PAGE || (ps & (ps - 1)) || bytes == 0)
            return ORC_E_CORRUPT;
        if (np != bytes / ps + (bytes % ps != 0) || nd > np || first != sum) return ORC_E_CORRUPT;
        if ((iflags & ORC_IMG_FULL) && nd != np) return ORC_E_CORRUPT;
        if (mode == ORC_MODE_HASH) any_hash = 1;
        for (uint64_t j = 0; j < nd; ++j) {
            if (first + j >= K) return ORC_E_CORRUPT;
            uint32_t id = rd32(ids + 4 * (first + j));
            if (id >= np) return ORC_E_CORRUPT;
            if (j > 0 && id <= rd32(ids + 4 * (first + j - 1))) return ORC_E_CORRUPT;
            if (has_hashes && mode != ORC_MODE_HASH && rd64(hashes + 8 * (first + j)) != 0)
                return ORC_E_CORRUPT;
        }
        sum += nd;
        pay += nd * ps;
    }
    if (sum != K || (!z && pay != payload) || any_hash != has_hashes) return ORC_E_CORRUPT;
    /* Compressed: one valid u16 size per 4 KiB unit, summing to the payload
     * length before its zero padding (readings Z2-Z3). */
    const uint8_t *zt = ids + tail_bytes_for(K, has_hashes);
    const uint64_t U = pay / ORC_UNIT;
    if (z) {
        if (total != ids_off + tail_bytes_for(K, has_hashes) + round_up(2 * U, 8)) return ORC_E_CORRUPT;
        uint64_t zb = 0;
        for (uint64_t u = 0; u < U; ++u) {
            uint64_t cs = (uint64_t)zt[2 * u] | ((uint64_t)zt[2 * u + 1] << 8);
            if (!z_size_ok(cs)) return ORC_E_CORRUPT;
            zb += cs;
        }
        for (uint64_t q = 2 * U; q < round_up(2 * U, 8); ++q)
            if (zt[q] != 0) return ORC_E_CORRUPT;
        if (round_up(zb, ORC_UNIT) != payload) return ORC_E_CORRUPT;
    }
    /* The table must describe the live registered set (reading Q11). */
    if (R != c->n) return ORC_E_MISMATCH;
    for (uint32_t k = 0; k < R; ++k) {
        const uint8_t *e = tab + 48 * (uint64_t)k;
        const orc_region *g = &c->r[k];
        if (rd32(e) != g->id || rd32(e + 4) != g->mode || rd64(e + 8) != g->bytes ||
            rd64(e + 16) != g->page_size || rd64(e + 24) != g->n_pages)
            return ORC_E_MISMATCH;
    }
    /* Compressed: decode every unit (a size that disagrees with its bitmap
     * is CORRUPT) before anything is written. */
    const uint8_t *pl = img + poff;
    if (z) {
        uint8_t *upay = (uint8_t *)malloc(pay ? pay : 1);
        uint64_t zb = 0;
        for (uint64_t u = 0; u < U; ++u) {
            uint64_t cs = (uint64_t)zt[2 * u] | ((uint64_t)zt[2 * u + 1] << 8);
            if (!orc_z_decode(img + poff + zb, cs, upay + u * ORC_UNIT)) {
                free(upay);
                return ORC_E_CORRUPT;
            }
            zb += cs;
        }
        pl = upay;
        *upay_out = upay;
    }
    /* CRUM_VERIFY: recompute the hash of every hash-mode slot. */
    if (flags & ORC_VERIFY) {
        uint64_t pbyte = 0;
        for (uint32_t k = 0; k < R; ++k) {
            const orc_region *g = &c->r[k];
            uint64_t first = rd64(tab + 48 * (uint64_t)k + 40), nd = rd64(tab + 48 * (uint64_t)k + 32);
            for (uint64_t j = 0; j < nd; ++j) {
                if (g->mode == ORC_MODE_HASH &&
                    orc_xxh3_64(pl + pbyte, g->page_size) != rd64(hashes + 8 * (first + j))) {
                    free(*upay_out);
                    *upay_out = NULL;
                    return ORC_E_CORRUPT;
                }
                pbyte += g->page_size;
            }
        }
    }
    return ORC_OK;
}

/* Write slot `slot` (page i of region g, payload bytes at src) back and commit
 * it: cur and mirror <- the logical bytes, table <- listed hash, force <- 0. */
static void restore_slot(orc_region *g, uint64_t i, const uint8_t *src, const uint8_t *hashes, uint64_t slot)
{
    uint64_t l = page_len(g, i);
    memcpy(g->cur + i * g->page_size, src, l);
    if (g->mode == ORC_MODE_COMPARE) memcpy(g->mirror + i * g->page_size, src, l);
    else if (g->mode == ORC_MODE_HASH) g->table[i] = rd64(hashes + 8 * slot);
    g->force[i] = 0;
}

/* Restart data movement (sec. 3.4; reading Q11): validate
 * everything first, then write each listed page's logical bytes back and
 * commit it (mirror <- slot / table <- listed hash, force <- 0). */
int orc_restore_scatter(orc_ctx *c, const uint8_t *img, uint64_t len, uint32_t flags,
                        orc_report *rep)
{
    if (!c || !img || (flags & ~ORC_VERIFY)) return ORC_E_INVAL;
    if (c->sess) return ORC_E_BUSY;
    uint8_t *upay;
    int st = validate_image(c, img, len, flags, &upay);
    if (st) return st;
    const uint32_t R = rd32(img + 12);
    const uint64_t K = rd64(img + 16), poff = rd64(img + 24), ids_off = rd64(img + 40), total = rd64(img + 48);
    const uint8_t *pl = upay ? upay : img + poff;
    const uint8_t *tab = img + 64;
    const uint8_t *ids = img + ids_off;
    const uint8_t *hashes = ids + round_up(4 * K, 8);
    /* Apply. */
    uint64_t pbyte = 0, dirty_bytes = 0, runs = 0, scanned = 0;
    for (uint32_t k = 0; k < R; ++k) {
        orc_region *g = &c->r[k];
        uint64_t first = rd64(tab + 48 * (uint64_t)k + 40), nd = rd64(tab + 48 * (uint64_t)k + 32);
        scanned += g->bytes;
        for (uint64_t j = 0; j < nd; ++j) {
            uint64_t i = rd32(ids + 4 * (first + j));
            restore_slot(g, i, pl + pbyte, hashes, first + j);
            dirty_bytes += page_len(g, i);
            if (j == 0 || rd32(ids + 4 * (first + j - 1)) + 1 != i) runs++;
            pbyte += g->page_size;
        }
    }
    if (rep) {
        rep->scanned_pages = total_pages(c);
        rep->scanned_bytes = scanned;
        rep->dirty_pages = K;
        rep->dirty_bytes = dirty_bytes;
        rep->dirty_runs = runs;
        rep->image_bytes = total;
    }
    free(upay);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Lazy restore: the paper's read-fault heuristic (sec. 4.2,           */
/* PAPER.md:783-793) applied to restart.  "For small shadow UVM        */
/* regions, it reads in all of the data ... for a read fault on a      */
/* large shadow UVM region, it starts off by only reading the data for */
/* just one page containing the faulting address.  On subsequent read  */
/* faults on the same region ... we exponentially increase (by powers  */
/* of 2) the number of pages read in."  Readings L1-L3:    */
/* small = at most 8 pages; the window starts at the faulting page and */
/* is clamped at the region end; a fault on a page already read in is  */
/* no fault; the window stops doubling at 2^62.                        */
/* ------------------------------------------------------------------ */
#define ORC_SMALL_REGION_PAGES 8ull

int orc_restore_begin(orc_ctx *c, const uint8_t *img, uint64_t len, uint32_t flags)
{
    if (!c || !img || (flags & ~ORC_VERIFY)) return ORC_E_INVAL;
    if (c->sess) return ORC_E_BUSY;
    uint8_t *upay;
    int st = validate_image(c, img, len, flags, &upay);
    if (st) return st;
    orc_session *s = (orc_session *)calloc(1, sizeof *s);
    s->img = img;
    s->upay = upay;
    s->present = (uint8_t **)calloc(c->n ? c->n : 1, sizeof(uint8_t *));
    s->window = (uint64_t *)calloc(c->n ? c->n : 1, sizeof(uint64_t));
    for (uint32_t k = 0; k < c->n; ++k) {
        s->present[k] = (uint8_t *)calloc(c->r[k].n_pages, 1);
        s->window[k] = 1;
    }
    s->written = (uint8_t *)calloc(rd64(img + 16) + 1, 1);
    c->sess = s;
    return ORC_OK;
}

/* Table entry k of the session's image: slots [first, first+nd), page size ps. */
static void entry_of(const uint8_t *img, uint32_t k, uint64_t *first, uint64_t *nd)
{
    *nd = rd64(img + 64 + 48 * (uint64_t)k + 32);
    *first = rd64(img + 64 + 48 * (uint64_t)k + 40);
}

/* Byte offset inside the payload of slot `slot` of table entry k. */
static uint64_t slot_payload_offset(const orc_ctx *c, const uint8_t *img, uint32_t k, uint64_t slot)
{
    uint64_t off = 0, first, nd;
    for (uint32_t q = 0; q < k; ++q) {
        entry_of(img, q, &first, &nd);
        off += nd * c->r[q].page_size;
    }
    entry_of(img, k, &first, &nd);
    return off + (slot - first) * c->r[k].page_size;
}

/* Write slot `slot` of the session's image (page i of region k) back. */
static void session_restore_slot(orc_ctx *c, uint32_t k, uint64_t i, uint64_t slot)
{
    const uint8_t *img = c->sess->img;
    const uint64_t K = rd64(img + 16), poff = rd64(img + 24), ids_off = rd64(img + 40);
    const uint8_t *hashes = img + ids_off + round_up(4 * K, 8);
    const uint8_t *pl = c->sess->upay ? c->sess->upay : img + poff;
    restore_slot(&c->r[k], i, pl + slot_payload_offset(c, img, k, slot), hashes, slot);
    c->sess->written[slot] = 1;
}

/* A read fault on page `page` of region `id`. */
int orc_restore_fetch(orc_ctx *c, uint32_t id, uint64_t page, uint64_t *covered, uint64_t *restored)
{
    if (!c || !c->sess || !covered || !restored) return ORC_E_INVAL;
    uint32_t k = 0;
    while (k < c->n && c->r[k].id != id) ++k;
    if (k == c->n) return ORC_E_NOREGION;
    orc_region *g = &c->r[k];
    if (page >= g->n_pages) return ORC_E_RANGE;
    orc_session *s = c->sess;
    *covered = 0;
    *restored = 0;
    if (s->present[k][page]) return ORC_OK;   /* already read in: no fault */
    uint64_t lo, hi;
    if (g->n_pages <= ORC_SMALL_REGION_PAGES) {
        lo = 0;                                /* small region: all of it */
        hi = g->n_pages;
    } else {
        lo = page;                             /* window pages from the faulting one */
        hi = g->n_pages - page < s->window[k] ? g->n_pages : page + s->window[k];
        if (s->window[k] < (1ull << 62)) s->window[k] *= 2;
    }
    const uint8_t *ids = s->img + rd64(s->img + 40);
    uint64_t first, nd;
    entry_of(s->img, k, &first, &nd);
    for (uint64_t i = lo; i < hi; ++i) {
        if (s->present[k][i]) continue;
        s->present[k][i] = 1;
        (*covered)++;
        for (uint64_t j = 0; j < nd; ++j) {    /* is page i listed in the image? */
            if (rd32(ids + 4 * (first + j)) == i) {
                session_restore_slot(c, k, i, first + j);
                (*restored)++;
                break;
            }
        }
    }
    return ORC_OK;
}

/* Close the session: every slot not yet written is written now. */
int orc_restore_end(orc_ctx *c, orc_report *rep)
{
    if (!c || !c->sess) return ORC_E_INVAL;
    orc_session *s = c->sess;
    const uint8_t *ids = s->img + rd64(s->img + 40);
    uint64_t dirty_bytes = 0, runs = 0, scanned = 0;
    for (uint32_t k = 0; k < c->n; ++k) {
        uint64_t first, nd;
        entry_of(s->img, k, &first, &nd);
        scanned += c->r[k].bytes;
        for (uint64_t j = 0; j < nd; ++j) {
            uint64_t i = rd32(ids + 4 * (first + j));
            if (!s->written[first + j]) session_restore_slot(c, k, i, first + j);
            dirty_bytes += page_len(&c->r[k], i);
            if (j == 0 || rd32(ids + 4 * (first + j - 1)) + 1 != i) runs++;
        }
    }
    if (rep) {
        rep->scanned_pages = total_pages(c);
        rep->scanned_bytes = scanned;
        rep->dirty_pages = rd64(s->img + 16);
        rep->dirty_bytes = dirty_bytes;
        rep->dirty_runs = runs;
        rep->image_bytes = rd64(s->img + 48);
    }
    for (uint32_t k = 0; k < c->n; ++k) free(s->present[k]);
    free(s->present);
    free(s->window);
    free(s->written);
    free(s->upay);
    free(s);
    c->sess = NULL;
    return ORC_OK;
}

/* Introspection for tests: copies of the force bits, hash table, mirror. */
int orc_get_force(orc_ctx *c, uint32_t id, uint8_t *out)
{
    orc_region *g = c ? find(c, id) : NULL;
    if (!g) return ORC_E_NOREGION;
    memcpy(out, g->force, g->n_pages);
    return ORC_OK;
}
int orc_get_hashes(orc_ctx *c, uint32_t id, uint64_t *out)
{
    orc_region *g = c ? find(c, id) : NULL;
    if (!g) return ORC_E_NOREGION;
    if (g->mode != ORC_MODE_HASH) return ORC_E_INVAL;
    memcpy(out, g->table, g->n_pages * sizeof(uint64_t));
    return ORC_OK;
}
int orc_get_mirror(orc_ctx *c, uint32_t id, uint8_t *out)
{
    orc_region *g = c ? find(c, id) : NULL;
    if (!g) return ORC_E_NOREGION;
    if (g->mode != ORC_MODE_COMPARE) return ORC_E_INVAL;
    memcpy(out, g->mirror, g->bytes);
    return ORC_OK;
}
int orc_page_hash(orc_ctx *c, uint32_t id, uint64_t i, uint64_t *out)
{
    orc_region *g = c ? find(c, id) : NULL;
    if (!g) return ORC_E_NOREGION;
    if (i >= g->n_pages) return ORC_E_RANGE;
    *out = page_hash(g, i);
    return ORC_OK;
}
