"""Test-only stand-in for the slab pass kernels (csrc/slab_kernels.cuh) on CPU
torch tensors, written with the oracle's numpy arithmetic. It lets the
distributed driver (paper_2006_10509_b200/slab.py: layout, corner turns,
all-to-all, sum reduction, cancel consensus) run under a real multi-process
gloo group without a GPU. Never used by the product path."""

import numpy as np
import torch

from oracle import cgh_oracle as O
from paper_2006_10509_b200.slab import SLAB_FINAL, SLAB_GS, SLAB_HOLO, SLAB_INIT, SLAB_INV, from_segments, to_segments


class NumpyOps:
    def __init__(self, cfg, n, world, rank):
        self.cfg, self.N, self.G, self.rank = cfg, n, world, rank
        self.R = n // world
        self.line0 = rank * self.R
        self.n_states = len(O.state_table(cfg.slm))
        fres = cfg.propagation.kind == "fresnel"
        self.q = O.quadratic_phase((n, n), cfg.propagation) if fres else None
        self.tgt = self.beam = None

    def empty(self, shape, kind="c"):
        dt = {"c": torch.complex128, "f64": torch.float64,
              "idx": torch.uint8 if self.n_states <= 256 else torch.int32}[kind]
        return torch.empty(shape, dtype=dt)

    def upload(self, arr, kind="c"):
        return torch.from_numpy(np.array(arr, dtype=np.complex128 if kind == "c" else None))

    def set_local(self, tgt, beam):
        self.tgt = np.array(tgt)
        self.beam = None if beam is None else np.array(beam)

    def transpose(self, src, dst):
        dst.copy_(src.transpose(1, 2))

    def _rows(self, data):
        return from_segments(data.numpy()).copy()

    def _store(self, data, rows):
        data.copy_(torch.from_numpy(np.ascontiguousarray(to_segments(rows))))

    def _snap(self, h, quantize, idx):
        if not quantize:
            return h
        k = O.nearest_state_index(h, self.cfg.slm)
        if idx is not None:
            idx.copy_(torch.from_numpy(k.astype(idx.numpy().dtype)))
        return O.state_table(self.cfg.slm)[k]

    def run(self, mode, data, gp=None, quantize=0, idx=None, sums=None):
        n, r0, r1 = self.N, self.line0, self.line0 + self.R
        beam = self.beam if self.beam is not None else 1.0
        q = None if self.q is None else self.q[r0:r1]
        if mode == SLAB_INIT:
            bg = np.random.PCG64()
            m = (1 << 64) - 1
            st = bg.state
            st["state"] = {"state": (gp.rng.state_hi << 64) | gp.rng.state_lo,
                           "inc": (gp.rng.inc_hi << 64) | gp.rng.inc_lo}
            st["has_uint32"], st["uinteger"] = gp.rng.has_uint32, gp.rng.uinteger
            bg.state = st
            bg.advance(r0 * n)
            u = np.random.Generator(bg).random((self.R, n))
            h = self._snap(beam * np.exp(1j * 2.0 * np.pi * u), quantize, idx)
            if q is not None:
                h = h * q
            self._store(data, np.fft.fft(h, axis=1))
            del m
            return
        x = self._rows(data)
        if mode == SLAB_HOLO:
            x = np.fft.ifft(x, axis=1) * n
            if q is not None:
                x = x * np.conj(q)
            mag = np.abs(x)
            h = np.where(mag > 0, beam * x / np.where(mag > 0, mag, 1.0), beam + 0j)
            h = self._snap(h, quantize, idx)
            if q is not None:
                h = h * q
            self._store(data, np.fft.fft(h, axis=1))
        elif mode == SLAB_INV:
            self._store(data, np.fft.ifft(x, axis=1) * n / n)
        else:
            rep = np.fft.fft(x, axis=1) / n
            rr = np.abs(rep)
            tt = self.tgt
            inside = ~np.signbit(tt)
            d = rr - tt
            s = [np.sum((d * d)[inside]), np.sum((rr * rr)[inside]), np.sum((rr * d)[inside]), np.sum(rr * rr)]
            sums.copy_(torch.tensor(s, dtype=torch.float64))
            if mode == SLAB_GS:
                want = np.clip(tt + self.cfg.feedback_gain * (tt - rr), 0.0, None)
                scale = np.where(rr > 0, want / np.where(rr > 0, rr, 1.0), 0.0)
                out = np.where(inside, np.where(rr > 0, rep * scale, want + 0j), rep)
                self._store(data, np.fft.ifft(out, axis=1) * n)
            assert mode in (SLAB_GS, SLAB_FINAL)

    def sync(self):
        pass
