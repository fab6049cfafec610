"""B200-native hot path of SAGA (arXiv 2605.00528): trace-driven KV-cache policy evaluation.

The compute path is libsaga.so (hand-written sm_100a CUDA behind the C ABI of include/saga.h);
`saga` is its ctypes binding and `pipeline` runs one pass of the hot path.  Import of `saga`
fails loudly when the extension is not built -- there is no CPU fallback.
"""
__all__ = ["saga", "pipeline"]
