"""B200-native QFactor-Sample instantiation (arXiv 2405.12866).

The product is the C-ABI library ``paper_2405_12866_b200/libqfs.so`` (see
``include/qfs.h``); ``paper_2405_12866_b200.qfs`` is its thin ctypes binding.
``paper_2405_12866_b200.inputs`` holds the seeded synthetic input generators.
"""
