"""B200-native Coded-InvNet coded-inference hot path (arXiv 2106.06445).

The compute lives in libcodedinv.so (hand-written sm_100a CUDA behind the C ABI in
include/codedinv.h); `codedinv` is its ctypes binding.  Importing `codedinv` fails
loudly if the library is not built.
"""
__all__ = ["codedinv", "build"]
