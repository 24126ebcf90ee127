"""Test helper: the same seeded regions registered with the CPU oracle (host
numpy buffers) and with libcrum.so (device tensors), kept in lock step.
Imports the oracle (test infrastructure) and the product binding side by side
-- they share nothing but the synth/ input recipe."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import oracle
from paper_1808_00117_b200 import crum


class Pair:
    def __init__(self, specs, S, chunk_bytes: int = 0, misalign: int = 0, device_writer: bool = True,
                 flags: int = 0, **ctx_kw):
        """specs: list of (nbytes, page_size, mode); flags: crum_config flags
        (kernel-path variants: CFG_NO_GRAPH, CFG_FUSED)."""
        self.specs = specs
        self.S = S
        self.o = oracle.Oracle()
        self.g = crum.Context(0, chunk_bytes=chunk_bytes, flags=flags, **ctx_kw)
        self.host, self.dev, self.rid_o, self.rid_g = [], [], [], []
        self._backing = []
        self.device_writer = device_writer
        for r, (nb, P, mode) in enumerate(specs):
            h = oracle.aligned_empty(nb)
            synth.fill_region(h, S, r)
            back = torch.empty(nb + misalign + 256, dtype=torch.uint8, device="cuda")
            d = back[misalign:misalign + nb]
            crum.synth_fill(d, nb, S, r)
            self.host.append(h)
            self.dev.append(d)
            self._backing.append(back)
            self.rid_o.append(self.o.register(h, P, mode))
            self.rid_g.append(self.g.register_region(d, nb, P, mode, keep=back))
        torch.cuda.synchronize()

    @property
    def N(self):
        return sum(synth.n_pages(nb, P) for nb, P, _ in self.specs)

    def write(self, epoch: int, d: float, touch: bool = False):
        """Application epoch: the same pages rewritten on host and device."""
        for r, (nb, P, _) in enumerate(self.specs):
            pages = synth.choose_dirty(self.S, epoch, r, synth.n_pages(nb, P), d)
            synth.apply_writer(self.host[r], P, pages, self.S, epoch, r, touch=touch)
            if self.device_writer:
                dp = torch.from_numpy(pages.astype(np.uint32)).cuda()
                crum.synth_write_pages(self.dev[r], nb, P, dp, len(pages), self.S, epoch, r, touch)
            else:
                self.dev[r].copy_(torch.from_numpy(self.host[r]))
        torch.cuda.synchronize()

    def regions_equal(self) -> bool:
        return all(np.array_equal(d.cpu().numpy(), h) for d, h in zip(self.dev, self.host))

    def oracle_flags(self) -> np.ndarray:
        return np.concatenate([self.o.detect(r) for r in self.rid_o]) if self.rid_o else np.zeros(0, np.uint8)

    def shadows_equal(self) -> bool:
        for (nb, P, mode), ro, rg in zip(self.specs, self.rid_o, self.rid_g):
            n = synth.n_pages(nb, P)
            if not np.array_equal(self.o.force_bits(ro), self.g.debug_export(rg, crum.EXPORT_FORCE, n)):
                return False
            if mode == crum.MODE_HASH:
                if not np.array_equal(self.o.hashes(ro), self.g.debug_export(rg, crum.EXPORT_HASHES, n)):
                    return False
            elif mode == crum.MODE_TRACKED:
                continue  # no snapshot: the force bits are the whole state
            else:
                if not np.array_equal(self.o.mirror(ro), self.g.debug_export(rg, crum.EXPORT_MIRROR, nb)):
                    return False
        return True
