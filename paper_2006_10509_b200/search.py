"""Host side of the SA / DBS runners (device kernels in csrc/search.cu)."""

from __future__ import annotations


def sa_call(cfg, target, illumination, progress, cancel, audit):
    raise NotImplementedError("SA device path lands in the next milestone")


def dbs_call(cfg, target, illumination, progress, cancel, audit):
    raise NotImplementedError("DBS device path lands in the next milestone")
