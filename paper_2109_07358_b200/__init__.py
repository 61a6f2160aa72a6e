"""B200-native fast fermion sampling (arXiv 2109.07358): CUDA hot path behind a C ABI.

Importing the package is cheap (no CUDA library load); `paper_2109_07358_b200.ffs` loads
libffs.so on first use and raises if it is missing — there is no CPU fallback.
"""
__all__ = ["ffs", "inputs", "build"]
