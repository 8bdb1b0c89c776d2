"""B200-native drop-in for the hologram-generation hot path of cghkit (HoloGen, arXiv 2006.10509).

Modules mirror the reference package layout (``cghkit.algorithms``,
``cghkit.propagation``, ``cghkit.slm``, ``cghkit.errors``, ``cghkit.kernels``,
``cghkit.image.rect_mask``) so ``import paper_2006_10509_b200 as cghkit``
style substitution works; compute runs in ``libcghb200.so`` (sm_100a CUDA).
"""

__version__ = "0.1.0"
