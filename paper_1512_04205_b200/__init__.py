"""cdmd-b200: B200-native (sm_100a) hot path of compressed DMD (arXiv 1512.04205).

    from paper_1512_04205_b200 import cdmd      # ctypes binding of libcdmd.so

The package never imports the test oracle (``oracle/``); without the built CUDA
library ``import paper_1512_04205_b200.cdmd`` raises ImportError.
"""

__all__ = ["cdmd", "build"]
