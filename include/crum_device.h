/*
 * crum_device.h -- device-side dirty marking for CRUM_MODE_TRACKED regions
 * (include in application CUDA code).
 *
 * Alg. 1 of the paper marks a page dirty when the application writes it
 * ("Page Fault ... else MarkPageAsDirty()").  GPU stores
 * cannot fault, so a kernel that writes a TRACKED region marks the pages it
 * wrote itself:
 *
 *     crum_tracker t;  crum_region_tracker(ctx, region_id, &t);   // host
 *     ...
 *     my_kernel<<<...>>>(..., t);
 *     __device__: x[i] = v;  crum_mark_write(t, i * sizeof(x[0]), sizeof(x[0]));
 *
 * Marking is idempotent (plain byte stores of 1), so any number of threads may
 * mark the same page.  The next crum_sync_shadow / crum_checkpoint_gather on a
 * stream ordered after the kernel lists exactly the marked pages.
 */
#ifndef CRUM_DEVICE_H
#define CRUM_DEVICE_H

#include "crum.h"

#ifdef __CUDACC__
static __device__ __forceinline__ void crum_mark_write(crum_tracker t, uint64_t offset, uint64_t len) {
    if (len == 0 || offset >= t.bytes) return;
    uint64_t last = offset + len - 1;
    if (last >= t.bytes) last = t.bytes - 1;
    for (uint64_t i = offset >> t.log2_page; i <= (last >> t.log2_page); ++i) t.force[i] = 1;
}

/* Whole page i (region-local index). */
static __device__ __forceinline__ void crum_mark_page(crum_tracker t, uint64_t i) {
    if (i <= ((t.bytes - 1) >> t.log2_page)) t.force[i] = 1;
}
#endif

#endif /* CRUM_DEVICE_H */
