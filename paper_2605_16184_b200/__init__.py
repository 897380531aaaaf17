# SPDX-License-Identifier: Apache-2.0
"""B200-native Asteria optimizer step (Shampoo / SOAP / KL-Shampoo).

The product is the in-tree shared library ``csrc/build/libasteria_b200.so``
(C-ABI: include/asteria_b200.h). ``runtime`` binds it with ctypes and raises
immediately if it is missing or no sm_100a device is present; there is no CPU
fallback.
"""
__all__ = ["abi", "runtime", "precond", "optimizer", "trace"]
