"""B200-native (sm_100a) randomized preconditioned CholeskyQR (arXiv 2111.11148).

The product is the C-ABI library libcqr.so (include/cqr.h) built from csrc/;
paper_2111_11148_b200.cholqr mirrors the reference's public API on top of it.
"""
