"""eDKM hot path on B200 (arXiv 2309.00964): DKM clustering on the <= 65,536 unique
16-bit weight patterns, forward and backward, behind the C ABI of libedkm.so.

Import ``paper_2309_00964_b200.edkm`` for the binding; ``synth`` holds the
seeded input generators; ``dist`` the multi-process orchestration.
"""
__all__ = ["edkm", "synth", "dist", "build"]
