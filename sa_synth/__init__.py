"""Seeded synthetic protein-family workloads (BASELINE.json ``configs``).

This package is shared INPUT tooling: both the CPU oracle (``oracle/``) and the
CUDA path read its output.  It holds none of the method's arithmetic (no k-mer
counting, no similarity, no ranking, no partitioning) -- only the random
generation of sequences, which stands in for the paper's Rose-generated and
Pfam workloads, none of which exist here.
"""
from .generator import CONFIGS, Dataset, WorkloadConfig, generate, generate_config  # noqa: F401
