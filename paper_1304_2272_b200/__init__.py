"""B200-native GLS hot path of arXiv 1304.2272 (drop-in for the reference package ``gwasgls``).

Modules mirror the reference's namespace: ``kernel`` (numerical core), ``fileio`` (formats and
async block agents), ``pipeline`` (in-core / out-of-core engines), ``shard`` (SNP-sharded
multi-GPU engine) and ``datagen`` (BASELINE generator).  Arithmetic runs in the sm_100a library
``libgwasgls_b200.so`` through the C-ABI of ``include/gwasgls_b200.h``.
"""

__version__ = "0.1.0"

from . import errors  # noqa: F401
