"""B200-native (sm_100a) shifted-Laplacian multigrid + FGMRES for the acoustic
Helmholtz equation (arXiv 2511.16808).  The compute path lives in
``csrc/`` (CUDA kernels behind the C-ABI of ``include/hmg.h``, built into
``libhmg.so``); ``hmg.py`` is the thin ctypes binding.  Importing this package
does not load the library; ``paper_2511_16808_b200.hmg`` does.
"""
__all__ = ["media", "hmg"]
