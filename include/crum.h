/*
 * crum.h -- C ABI of the B200-native shadow-page synchronisation library
 * (libcrum.so), the data-parallel hot path of CRUM (arXiv 1808.00117).
 *
 * The calls follow the paper's statement of the problem:
 *   Alg. 1 "Shadow page synchronization algorithm":
 *     - "CUDA Create UVM region": CreateShadowPage, all pages dirty
 *                           -> crum_register_region
 *     - "Page Fault ... MarkPageAsDirty()"
 *                                                       -> crum_mark_dirty and
 *       content-based detection inside every sync/gather (reading Q1)
 *     - "CUDA call: if hasDirtyPages: SendDataToRealPages(); ClearDirtyPages()"
 *                           -> crum_sync_shadow
 *   sec. 3.4 checkpoint drain: "for all the active CUDA-MALLOC and CUDA-UVM
 *     memory regions, data is read in from the GPU to the host"
 *                                                       -> crum_checkpoint_gather
 *   sec. 3.4 restart: "transfers the data into the actual CUDA and CUDA-UVM
 *     regions"                       -> crum_restore_scatter
 *
 * Conventions (all functions):
 *   - Return int: CRUM_OK (0) or a negative crum_status.  No exceptions cross
 *     the ABI, nothing calls exit().  On any error other than CRUM_E_CUDA no
 *     state changes: registry, snapshots, hash tables and force bits are
 *     untouched; a failed gather commits nothing; a rejected restore writes
 *     nothing.  CRUM_E_CUDA is sticky: it poisons the context (every later
 *     call on it returns CRUM_E_CUDA); crum_last_error_detail() says why.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Work is enqueued after all prior work on `stream`: that is the
 *     quiescence point, the analog of the paper's cudaDeviceSynchronize drain
 *     (PAPER.md:545).  Writers on other streams during a call are undefined
 *     behaviour.  The library keeps no stream handle after a call returns.
 *   - Device pointers are plain CUDA device (or managed) addresses on the
 *     context's device; host pointers are ordinary process addresses.
 *   - A context is single-threaded (one thread at a time per context).
 */
#ifndef CRUM_H
#define CRUM_H

#include <stddef.h>
#include <stdint.h>

#ifndef CRUM_API
#if defined(__GNUC__)
#define CRUM_API __attribute__((visibility("default")))
#else
#define CRUM_API
#endif
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CRUM_ABI_VERSION 1

/* Status codes. */
enum crum_status {
    CRUM_OK = 0,
    CRUM_E_INVAL = -1,     /* null pointer, bytes == 0, bad page size / mode / flags, misaligned ptr */
    CRUM_E_OVERLAP = -2,   /* new range overlaps a live region ("Overlap") */
    CRUM_E_NOREGION = -3,  /* unknown region id */
    CRUM_E_RANGE = -4,     /* crum_mark_dirty range outside the region */
    CRUM_E_NOMEM = -5,     /* device or pinned host allocation failed */
    CRUM_E_CAPACITY = -6,  /* image buffer too small; report->image_bytes = required size */
    CRUM_E_CORRUPT = -7,   /* bad magic/version/CRC/sizes/ids, or a hash mismatch under CRUM_VERIFY */
    CRUM_E_MISMATCH = -8,  /* image region table != live registered set */
    CRUM_E_BUSY = -9,      /* gather into an image whose persist is still in flight */
    CRUM_E_DEVICE = -10,   /* ptr not accessible from the context's device; no such device */
    CRUM_E_CUDA = -11,     /* underlying CUDA error (sticky) */
    CRUM_E_IO = -12        /* file I/O failed (persist / load); detail via crum_last_error_detail */
};

/* Per-region dirty-detection mode (reading Q1/Q8). */
typedef enum {
    CRUM_MODE_COMPARE = 0,   /* device byte mirror of the region, per-page compare */
    CRUM_MODE_HASH_XXH3 = 1, /* 8 B per page: XXH3-64 (seed 0) of the zero-padded page slot */
    CRUM_MODE_TRACKED = 2    /* no shadow: a page is dirty iff it was marked since its last commit
                                (Alg. 1 MarkPageAsDirty on writes) -- by
                                crum_mark_dirty[_pages] or, inside application kernels, by
                                crum_mark_write() of include/crum_device.h.  Unmarked writes are
                                not captured. */
} crum_mode;

/* Call flags. */
enum {
    CRUM_FULL = 1u << 0,    /* gather: list every page (the paper's full drain) */
    CRUM_VERIFY = 1u << 1,  /* restore: recompute and check every hash-mode slot before writing */
    CRUM_COMPRESS = 1u << 2 /* gather: compressed image (readings Z1-Z2; the paper's
                               in-memory compression before writing):
                               every 4 KiB payload unit is encoded on the GPU -- 1024 LE u32
                               words, word j predicted by word j-2; 0 mispredicted words -> 0
                               bytes; else a 128-byte bitmap + the mispredicted words if shorter
                               than 4096, else raw -- and only encoded bytes cross the host link
                               (the encoder stores straight into the mapped pinned image).
                               Restore decodes transparently.  Image flag bit2; the tail gains a
                               u16 encoded size per unit after the hashes (padded to 8). */
};

typedef struct crum_ctx crum_ctx;     /* one per (process, CUDA device) */
typedef struct crum_image crum_image; /* library-owned pinned host buffer holding one image */

/* Per-context configuration (SURVEY.md sec. 8(b)/sec. 5: chunk bytes, pinned
 * pool bytes, NUMA node, flags).  Every tuning choice of the library lives
 * here, per context -- the library reads no environment variables. */
typedef struct {
    uint64_t chunk_bytes;       /* host-link pipeline chunk (0 = 64 MiB); multiple of 4096 */
    uint64_t pinned_pool_bytes; /* 0: every crum_image is its own pinned allocation.  > 0: one
                                   pinned, device-mapped pool of this many bytes (multiple of
                                   4096) is reserved at crum_create on the images' NUMA node and
                                   images are carved from it (first fit, 4 KiB granules, freed
                                   ranges coalesce); an image that does not fit gets its own
                                   allocation.  Pinning is slow (seconds per 8 GiB), the pool
                                   pays it once. */
    int32_t numa_node;          /* host node of pinned images and the pool:
                                   CRUM_NUMA_AUTO (-1): the node of the GPU's PCIe root on a
                                     multi-node host, default placement otherwise;
                                   CRUM_NUMA_DEFAULT (-2): default placement (cudaHostAlloc);
                                   >= 0: that node (anonymous mmap + mbind + cudaHostRegister). */
    uint32_t flags;             /* CRUM_CFG_* below */
} crum_config;

enum { CRUM_NUMA_AUTO = -1, CRUM_NUMA_DEFAULT = -2 };

/* Fill *cfg with the defaults (chunk 64 MiB, no pool, CRUM_NUMA_AUTO, no
 * flags) -- note that a zero-filled struct means NUMA node 0.  Passing
 * cfg = NULL to crum_create is the same as these defaults.
 * Errors: INVAL (null cfg). */
CRUM_API int crum_config_init(crum_config *cfg);

/* crum_config.flags.
 *   CRUM_CFG_TIMING   record CUDA events around the phases of EVERY call (also
 *                     asynchronous ones), so crum_last_report can return phase
 *                     times without the call itself waiting.  The one-launch
 *                     small-footprint kernel times itself instead (globaltimer
 *                     stamps, see CRUM_PATH_SMALL).  Calls that return a report
 *                     (pinned-image gathers, synchronous device gathers) time
 *                     themselves with or without this flag.
 *   CRUM_CFG_NO_GRAPH never replay a captured CUDA graph for asynchronous device
 *                     gathers (every launch is enqueued directly).
 *   CRUM_CFG_FUSED    device-image gathers of a context whose regions are all
 *                     COMPARE with pages <= 64 KiB run the single-pass kernel
 *                     (detect + compaction + gather + commit in one launch).
 *   CRUM_CFG_TRACE    print the host pipeline's per-range times to stderr.
 *   CRUM_CFG_NO_MAPPED pinned-image gathers never take the mapped-store range
 *                     pipeline (CRUM_PATH_MAPPED); every payload goes through the
 *                     device ring and D2H copies. */
enum {
    CRUM_CFG_TIMING = 1u << 0,
    CRUM_CFG_NO_GRAPH = 1u << 1,
    CRUM_CFG_FUSED = 1u << 2,
    CRUM_CFG_TRACE = 1u << 3,
    CRUM_CFG_NO_MAPPED = 1u << 4
};

/* Outcome of a sync / gather / restore.  Times are CUDA-event milliseconds
 * on the call's stream (0 when not measured). */
typedef struct {
    uint64_t scanned_pages;  /* N = sum of n_r over live regions */
    uint64_t scanned_bytes;  /* F = sum of B_r */
    uint64_t dirty_pages;    /* K (pages listed / committed / restored) */
    uint64_t dirty_bytes;    /* sum of logical lengths of those pages */
    uint64_t dirty_runs;     /* maximal runs of consecutive page indices, summed over regions */
    uint64_t image_bytes;    /* image length (gather, restore); required size on CRUM_E_CAPACITY */
    double t_detect_ms;      /* A1: detect */
    double t_compact_ms;     /* A2: compact + image metadata */
    double t_gather_ms;      /* A3: gather + commit (restore: scatter + commit) */
    double t_copy_ms;        /* A4: host-link copy (D2H for gather, H2D for restore) */
    double t_total_ms;       /* whole call, first enqueue to completion */
    uint32_t path;           /* bit0 CRUM_PATH_FUSED: single-pass detect+compact+gather kernel ran
                                (t_detect_ms then covers all three, t_gather_ms is 0);
                                bit1 CRUM_PATH_COMPRESSED: compressed gather (t_compact_ms includes
                                the encoded-size pass, t_gather_ms is encode + commit, including
                                the host-link stores for a pinned image; t_copy_ms is 0);
                                bit2 CRUM_PATH_SMALL (with bit0): the one-launch small-footprint
                                kernel, which also writes the metadata; with CRUM_CFG_TIMING it
                                times itself (globaltimer, first CTA in -> last CTA out), so
                                t_detect_ms = t_total_ms = the kernel, and no events are recorded
                                around it;
                                bit3 CRUM_PATH_MAPPED: pinned gather whose kernels stored the
                                payload and metadata straight into the image through its mapped
                                address, range by range with no host wait between ranges (small
                                payloads); t_copy_ms is then the span of those stores */
    uint32_t reserved;
} crum_report;

enum { CRUM_PATH_FUSED = 1u << 0, CRUM_PATH_COMPRESSED = 1u << 1, CRUM_PATH_SMALL = 1u << 2, CRUM_PATH_MAPPED = 1u << 3 };

/* ---------------------------------------------------------------------------
 * Context.  crum_create binds to CUDA device `device` (cudaSetDevice is
 * called by every entry point).  cfg may be NULL (defaults).  Errors:
 * INVAL (null out / bad cfg), DEVICE (no such device), NOMEM, CUDA.
 * crum_destroy frees everything the library owns for this context (snapshots,
 * hash tables, scratch); images must be destroyed before their context.
 * ------------------------------------------------------------------------- */
CRUM_API int crum_create(int device, const crum_config *cfg, crum_ctx **out);
CRUM_API int crum_destroy(crum_ctx *ctx);

/* ---------------------------------------------------------------------------
 * Alg. 1 "CUDA Create UVM region".  Registers the caller's
 * device/managed range [ptr, ptr+bytes) split into pages of page_size bytes
 * (the last page may be partial: logical length B - i*P, Q7) and
 * creates its shadow: a device byte mirror (COMPARE) or an 8 B/page hash
 * table (HASH_XXH3).  Every page starts force-dirty ("all the pages in the
 * regions are marked as dirty"), so the first sync/gather
 * lists all n = ceil(bytes/page_size) pages.
 * ptr may be device memory of the context's device, managed (UVM) memory, or
 * pinned host memory mapped at the same address (cudaHostAlloc under UVA):
 * host-resident pages are then read over the host link.
 * Preconditions: ptr 16-byte aligned, accessible from the context's device;
 * bytes > 0; page_size a power of two in [4096, 2 MiB]; n < 2^32 and the
 * context's total page count < 2^31; no overlap with a live region.
 * Ownership: the caller owns ptr and must keep it valid until unregister; the
 * library never frees or moves it.  Region ids start at 1, increase
 * monotonically and are never reused; id order is image order.
 * Errors: INVAL, DEVICE, OVERLAP, NOMEM, CUDA.
 * ------------------------------------------------------------------------- */
CRUM_API int crum_register_region(crum_ctx *ctx, void *ptr, uint64_t bytes, uint64_t page_size,
                         uint32_t mode, uint32_t *region_id_out);
CRUM_API int crum_unregister_region(crum_ctx *ctx, uint32_t region_id);

/* Batch form of crum_register_region for applications with many regions
 * (the paper's HPGMG-FV allocates thousands of 12-128 KB boxes):
 * registers descs[0..n) with ONE rebuild of the device descriptors instead of
 * n.  Each descriptor has crum_register_region's preconditions, ownership and
 * shadow; the new ids are consecutive, in descriptor order (so descriptor
 * order is image order).  Transactional: on any error no region is
 * registered and *failed_index_out (nullable) holds the index of the first
 * offending descriptor (UINT32_MAX when the error is not tied to one).
 * n == 0 is a no-op.  Errors: INVAL, DEVICE, OVERLAP (also between two
 * descriptors of the batch), NOMEM, CUDA. */
typedef struct {
    void *ptr;          /* region start (device / managed / UVA-mapped pinned host), 16-byte aligned */
    uint64_t bytes;     /* > 0 */
    uint64_t page_size; /* power of two in [4096, 2 MiB] */
    uint32_t mode;      /* CRUM_MODE_* */
    uint32_t reserved;  /* 0 */
} crum_region_desc;
CRUM_API int crum_register_regions(crum_ctx *ctx, uint32_t n, const crum_region_desc *descs,
                                   uint32_t *region_ids_out, uint32_t *failed_index_out);

/* Alg. 1 MarkPageAsDirty as an explicit call: sets the force
 * bit of every page overlapping [offset, offset+len).  len == 0 is a no-op.
 * Errors: NOREGION, RANGE (offset+len > bytes). */
CRUM_API int crum_mark_dirty(crum_ctx *ctx, uint32_t region_id, uint64_t offset, uint64_t len);

/* Stream-ordered batch marking: sets the force bit of page dev_pages[k]
 * (region-local page indices, a DEVICE array of n u32) for k < n, after all
 * prior work on `stream`.  Indices >= the region's page count are ignored.
 * Errors: NOREGION, INVAL (dev_pages NULL with n > 0), CUDA. */
CRUM_API int crum_mark_dirty_pages(crum_ctx *ctx, uint32_t region_id, const uint32_t *dev_pages, uint64_t n,
                                   void *stream);

/* Device-side marking handle of one region: application kernels call
 * crum_mark_write(tracker, offset, len) (include/crum_device.h) after writing
 * [offset, offset+len) of the region.  `force` points at the region's force
 * bits in device memory; it is invalidated by the next register/unregister on
 * the context (call crum_region_tracker again). */
typedef struct {
    uint8_t *force;     /* device pointer: one byte per page */
    uint64_t bytes;     /* region bytes */
    uint32_t log2_page; /* log2(page_size) */
    uint32_t reserved;
} crum_tracker;
CRUM_API int crum_region_tracker(crum_ctx *ctx, uint32_t region_id, crum_tracker *out);

/* ---------------------------------------------------------------------------
 * Alg. 1 "CUDA call" event: detect the dirty pages of every
 * live region (force bit, or bytes differ from the snapshot / XXH3 differs
 * from the stored hash), then commit them (snapshot <- current, force <- 0).
 * If dirty_pages_out is non-NULL the call waits and stores K; if NULL the call
 * is fully stream-asynchronous.  An immediate second sync returns 0.
 * ------------------------------------------------------------------------- */
CRUM_API int crum_sync_shadow(crum_ctx *ctx, void *stream, uint64_t *dirty_pages_out);

/* Upper bound on the image size when at most max_dirty_pages are listed
 * (pass UINT64_MAX for "every page"), plain or CRUM_COMPRESS (it includes the
 * 2 bytes per 4 KiB unit of a compressed image's unit-size table). */
CRUM_API int crum_image_required_bytes(crum_ctx *ctx, uint64_t max_dirty_pages, uint64_t *bytes_out);

/* Pinned host images, mapped into the device's address space.  On a host
 * with more than one NUMA node the pages are placed on the node of the
 * GPU's PCIe root (sysfs numa_node; anonymous mmap + mbind(MPOL_PREFERRED)
 * + cudaHostRegister), so the copy-out of SURVEY.md sec. 8(e) ("pinned
 * images must be NUMA-local to each GPU") never crosses the socket link;
 * otherwise, or if that fails, cudaHostAlloc.  crum_config.numa_node
 * overrides the node.  With crum_config.pinned_pool_bytes > 0 images are
 * carved from the context's pinned pool when they fit (the context must then
 * outlive its images).  crum_image_import copies `len` bytes into a
 * new image (for restart from a file).  crum_image_data exposes the buffer:
 * *data_out (host pointer, owned by the image), *len_out (valid image
 * length; 0 before the first gather), *capacity_out (may be NULL). */
CRUM_API int crum_image_create(crum_ctx *ctx, uint64_t capacity_bytes, crum_image **out);
CRUM_API int crum_image_import(crum_ctx *ctx, const void *bytes, uint64_t len, crum_image **out);
CRUM_API int crum_image_data(const crum_image *img, void **data_out, uint64_t *len_out, uint64_t *capacity_out);
CRUM_API int crum_image_destroy(crum_image *img);
/* *node_out = the NUMA node the image's pages were bound to, -1 for default
 * placement (single-node host, CRUM_NUMA_DEFAULT, or mbind refused by the
 * sandbox).  Errors: INVAL (null argument). */
CRUM_API int crum_image_numa_node(const crum_image *img, int *node_out);
/* The context's pinned pool (crum_config.pinned_pool_bytes): *bytes_out its
 * size (0: no pool), *in_use_out bytes currently carved out (4 KiB granules),
 * *largest_free_out the largest free extent, *images_out images living in it.
 * Any out pointer may be NULL.  Errors: INVAL (null ctx). */
CRUM_API int crum_pinned_pool_info(crum_ctx *ctx, uint64_t *bytes_out, uint64_t *in_use_out,
                                   uint64_t *largest_free_out, uint32_t *images_out);
/* *node_out = the host NUMA node of CUDA device `device`'s PCIe function, or
 * -1 when unknown or when the host has one node (callers use it to pin the
 * rank's host threads next to its GPU).  Errors: INVAL (null node_out),
 * DEVICE (no such device). */
CRUM_API int crum_device_numa_node(int device, int *node_out);

/* ---------------------------------------------------------------------------
 * Asynchronous ("forked") persistence, the paper's forked checkpoint
 * (sec. 3.3): once the GPU has been drained into the pinned
 * image, a writer thread stores it to `path` while the application goes on;
 * the pause is the gather alone.  While a persist is in flight the image is
 * busy: a gather into it returns CRUM_E_BUSY (SPEC.md:441
 * "ConcurrentCheckpoint"), so applications alternate two images; restoring
 * from it is allowed (the writer only reads it).
 *   crum_image_persist: start writing img[0, len) to path (created/truncated);
 *     flags: CRUM_PERSIST_FSYNC (fsync before completion); CRUM_PERSIST_DIRECT
 *     (O_DIRECT: the writer's bytes go from the pinned image to the device
 *     without a page-cache copy -- whole 4 KiB blocks, the file then
 *     truncated to the image length; a filesystem without O_DIRECT support
 *     makes the writer fail with CRUM_E_IO).  Errors: INVAL, BUSY.
 *   crum_image_persist_wait: wait for the writer; returns its outcome (OK or
 *     CRUM_E_IO); OK if none is in flight.
 *   crum_image_persist_busy: *busy_out = 1 while the writer runs.
 *   crum_image_load: new pinned image holding the file's bytes (restart from
 *     storage).  Errors: INVAL, IO, NOMEM.
 * crum_image_destroy waits for an in-flight writer first.
 * ------------------------------------------------------------------------- */
enum { CRUM_PERSIST_FSYNC = 1u << 0, CRUM_PERSIST_DIRECT = 1u << 1 };
CRUM_API int crum_image_persist(crum_image *img, const char *path, uint32_t flags);
CRUM_API int crum_image_persist_wait(crum_image *img);
CRUM_API int crum_image_persist_busy(const crum_image *img, int *busy_out);
CRUM_API int crum_image_load(crum_ctx *ctx, const char *path, crum_image **out);

/* ---------------------------------------------------------------------------
 * sec. 3.4 checkpoint drain as an incremental gather (DESIGN
 * readings Q5/Q12): detect (A1), compact the dirty ids in (region id, page
 * index) order (A2), gather those pages into the v1 image (A3; DESIGN.md
 * "Image format") and commit them, copying the image into `img` in pinned host
 * memory over the host link (A4): range by range through a device ring and
 * D2H copies, or -- small expected payloads, an image that holds a worst-case
 * image -- stored by the kernels through the image's device-mapped address
 * (CRUM_PATH_MAPPED).  flags: 0, CRUM_FULL, CRUM_COMPRESS.
 * Returns when the image is complete in host memory and the commit is done.
 * Errors: INVAL; CAPACITY (nothing committed; report->image_bytes = needed);
 * CUDA.  report may be NULL.
 * ------------------------------------------------------------------------- */
CRUM_API int crum_checkpoint_gather(crum_ctx *ctx, crum_image *img, void *stream, uint32_t flags,
                           crum_report *report_out);

/* Same, but the image is written into a caller-owned DEVICE buffer
 * [dev_image, dev_image+capacity) and never crosses the host link.
 * If report_out is NULL the call is stream-asynchronous and capacity must be
 * >= crum_image_required_bytes(ctx, UINT64_MAX) (else CAPACITY, checked on the
 * host before anything is enqueued); with a report the call waits, and an
 * image larger than capacity returns CAPACITY with nothing committed.
 * The image length is report_out->image_bytes (also header bytes 32..47). */
CRUM_API int crum_checkpoint_gather_device(crum_ctx *ctx, void *dev_image, uint64_t capacity, void *stream,
                                  uint32_t flags, crum_report *report_out);

/* ---------------------------------------------------------------------------
 * sec. 3.4 restart (reading Q11): validate the image
 * (magic, version, both CRC-32s, sizes, ids strictly ascending and in range,
 * table == live registered set), then write each listed page's logical bytes
 * back into its region and commit it (snapshot <- slot / table <- listed
 * hash, force <- 0).  flags: 0 or CRUM_VERIFY.  Pages not listed are left
 * alone, so image k restores state k onto state k-1.
 * Errors: INVAL, CORRUPT, MISMATCH (nothing written), CUDA.
 * ------------------------------------------------------------------------- */
CRUM_API int crum_restore_scatter(crum_ctx *ctx, const crum_image *img, void *stream, uint32_t flags,
                         crum_report *report_out);
CRUM_API int crum_restore_scatter_device(crum_ctx *ctx, const void *dev_image, uint64_t len, void *stream,
                                uint32_t flags, crum_report *report_out);

/* ---------------------------------------------------------------------------
 * Lazy restore with exponential prefetch: the paper's read-fault heuristic
 * (sec. 4.2: "for small shadow UVM regions, it reads in all
 * of the data ... for a read fault on a large shadow UVM region, it starts off
 * by only reading the data for just one page containing the faulting address.
 * On subsequent read faults on the same region ... we exponentially increase
 * (by powers of 2) the number of pages read in"), applied to restart.
 *
 * crum_restore_begin: every check of crum_restore_scatter (CRUM_VERIFY
 *   included), nothing written.  The image must stay alive and unchanged until
 *   crum_restore_end (gathers into it and crum_image_destroy return BUSY).
 *   While the session is open, register / unregister / sync / gather /
 *   restore / crum_destroy on ctx return CRUM_E_BUSY; crum_mark_dirty[_pages]
 *   and application writes to fetched pages are fine.  Errors: as
 *   crum_restore_scatter, plus BUSY (a session is already open).
 * crum_restore_fetch: the application is about to read page `page` of
 *   region `region_id` (a "read fault").  If the page is already present,
 *   nothing happens (*covered_out = 0).  Otherwise the fault's window is made
 *   present: the whole region if it has at most 8 pages, else pages
 *   [page, page + w) clamped at the region end, where w is 1 on the region's
 *   first fault and doubles after each fault (reading L1-L3).
 *   Pages of the window already present are skipped; image slots of the rest
 *   are written (region bytes + commit, as crum_restore_scatter) by kernels
 *   on `stream`, reading the pinned image in place.  *covered_out = pages newly
 *   present, *restored_out = image slots written (either may be NULL).
 *   Stream-asynchronous: wait on `stream` before reading the pages elsewhere.
 *   Errors: INVAL, NOREGION, RANGE (page >= n_r), CUDA.
 * crum_restore_end: writes every slot not written yet, waits, closes the
 *   session (always, even on error).  report_out (may be NULL) as
 *   crum_restore_scatter's (dirty_pages = K of the image).
 * Result: begin + any fetch sequence + end leaves regions, snapshots and
 * force bits exactly as crum_restore_scatter of the same image.
 * ------------------------------------------------------------------------- */
typedef struct crum_restore_session crum_restore_session;
CRUM_API int crum_restore_begin(crum_ctx *ctx, crum_image *img, void *stream, uint32_t flags,
                                crum_restore_session **out);
CRUM_API int crum_restore_fetch(crum_restore_session *session, uint32_t region_id, uint64_t page, void *stream,
                                uint64_t *covered_out, uint64_t *restored_out);
CRUM_API int crum_restore_end(crum_restore_session *session, void *stream, crum_report *report_out);

/* Report of the most recent sync / gather / restore call on ctx: waits for
 * that call's work to finish, then fills counters and (if events were
 * recorded: a report was requested or CRUM_CFG_TIMING is set) phase times.
 * Errors: INVAL (null, or no call yet), CUDA. */
CRUM_API int crum_last_report(crum_ctx *ctx, crum_report *report_out);

/* Status text; thread-local detail of the last error on this thread. */
CRUM_API const char *crum_status_string(int status);
CRUM_API const char *crum_last_error_detail(void);

/* ---------------------------------------------------------------------------
 * Test/parity hooks (not on the hot path).
 * crum_debug_detect: run A1 over every live region WITHOUT committing and copy
 *   (force | changed) per page, in global page order (regions ascending), into
 *   host_flags[0..n) (n must equal the total page count).
 * crum_debug_export: copy a region's FORCE bits (u8 per page), HASHES (u64 per
 *   page, hash mode) or MIRROR (B bytes, compare mode) into host_buf (len must
 *   match exactly).
 * ------------------------------------------------------------------------- */
enum { CRUM_EXPORT_FORCE = 0, CRUM_EXPORT_HASHES = 1, CRUM_EXPORT_MIRROR = 2 };
CRUM_API int crum_debug_detect(crum_ctx *ctx, void *stream, uint8_t *host_flags, uint64_t n);
CRUM_API int crum_debug_export(crum_ctx *ctx, uint32_t region_id, int what, void *host_buf, uint64_t len);

/* Number of kernel launches this context has enqueued so far (bench evidence). */
CRUM_API uint64_t crum_launch_count(const crum_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* CRUM_H */
