/*
 * crum_synth.h -- seeded synthetic-input kernels exported by libcrum.so for
 * tests and bench.py (NOT part of the shadow-page method).  They implement
 * the counter-based recipe of synth/__init__.py
 * on the device, so multi-GiB footprints need not cross the host link:
 *
 *   content: u64 word j of region r = splitmix64(S ^ (r << 40) ^ (word_offset + j))
 *   writer : each listed page's logical words ^= splitmix64((S+2) ^ (epoch << 56)
 *            ^ (r << 40) ^ page) | 1   (touch != 0: only the page's last word)
 *
 * All pointers are device pointers; work is enqueued on `stream` (void* =
 * cudaStream_t).  Returns CRUM_OK or CRUM_E_INVAL / CRUM_E_CUDA.
 */
#ifndef CRUM_SYNTH_H
#define CRUM_SYNTH_H

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

CRUM_API int crum_synth_fill(void *dev_ptr, uint64_t bytes, uint64_t seed, uint64_t region_index,
                    uint64_t word_offset, void *stream);

CRUM_API int crum_synth_write_pages(void *dev_ptr, uint64_t bytes, uint64_t page_size,
                           const uint32_t *dev_pages, uint64_t n_pages, uint64_t seed,
                           uint64_t epoch, uint64_t region_index, int touch, void *stream);

/* Same writer for a CRUM_MODE_TRACKED region: each written page is also marked
 * through `tracker` (crum_region_tracker) with crum_mark_write() of
 * include/crum_device.h, inside the writer kernel -- the way an application
 * kernel marks what it writes. */
CRUM_API int crum_synth_write_pages_tracked(void *dev_ptr, uint64_t bytes, uint64_t page_size,
                                           const uint32_t *dev_pages, uint64_t n_pages, uint64_t seed,
                                           uint64_t epoch, uint64_t region_index, int touch,
                                           const void *tracker /* const crum_tracker* */, void *stream);

/* Many regions in one launch (a footprint of thousands of regions -- config 4
 * -- would otherwise cost one launch per region per epoch).  `regions` is a
 * HOST array of n descriptors (copied before the call returns); region i gets
 * exactly what crum_synth_fill(dev_ptr, bytes, seed, region_index, 0) /
 * crum_synth_write_pages(dev_ptr, bytes, page_size, dev_pages, n_pages, seed,
 * epoch, region_index, touch) give it (dev_pages: device u32 page list, may be
 * NULL when n_pages == 0).  Errors: INVAL (a null or unaligned pointer, a page
 * size that is 0 or not a multiple of 8), NOMEM, CUDA. */
typedef struct crum_synth_region {
    void *dev_ptr;
    uint64_t bytes;
    uint64_t page_size;        /* writer only */
    uint64_t region_index;
    const uint32_t *dev_pages; /* writer only */
    uint64_t n_pages;          /* writer only */
} crum_synth_region;
CRUM_API int crum_synth_fill_regions(const crum_synth_region *regions, uint64_t n, uint64_t seed, void *stream);
CRUM_API int crum_synth_write_regions(const crum_synth_region *regions, uint64_t n, uint64_t seed, uint64_t epoch,
                                      int touch, void *stream);

/* Streaming read of `bytes` (device buffer) between timed repetitions: evicts
 * L2 (writing dirty lines back outside the timed region), leaves it clean. */
CRUM_API int crum_synth_scrub(void *dev_ptr, uint64_t bytes, void *stream);

/* Bandwidth probe: 16-byte vectorised copy kernel (blocks <= 0: 8 per SM of a
 * 148-SM part).  dst/src may be device or mapped pinned host pointers, 16-byte
 * aligned, bytes a multiple of 16. */
CRUM_API int crum_probe_copy(void *dst, const void *src, uint64_t bytes, int blocks, void *stream);

/* Config-5 footprint: cudaMallocManaged of `bytes`; [0, device_bytes) gets
 * PreferredLocation = device (prefetched there), the rest PreferredLocation =
 * CPU + AccessedBy = device (prefetched to host), so GPU scans read it over
 * the host link without migrating it.  *out receives the managed pointer.
 * Errors: INVAL, DEVICE, NOMEM, CUDA.  Free with crum_synth_free_managed. */
CRUM_API int crum_synth_alloc_managed(void **out, uint64_t bytes, int device, uint64_t device_bytes);
CRUM_API int crum_synth_free_managed(void *p);

#ifdef __cplusplus
}
#endif

#endif /* CRUM_SYNTH_H */
