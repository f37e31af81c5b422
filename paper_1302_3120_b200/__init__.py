"""paper_1302_3120_b200 — B200-native hot path of fast CS-SAR imaging based on approximated
observation (arXiv 1302.3120): libcssar.so (CUDA, sm_100a) + a thin ctypes binding.

The product path has no CPU fallback and does not import oracle/."""
from .cssar import Plan, Group, pack_mask, load_library, nccl_unique_id, slab_rows, CssarError  # noqa: F401
from .batch import BatchRunner  # noqa: F401
