"""paper_1702_04458_b200 -- B200-native decentralized baseband processing.

Thin Python binding over ``libdbp.so`` (the C ABI declared in
``include/dbp.h``).  Importing the package does not load the CUDA library;
the first call does, and raises ``DbpError`` if the extension is missing or
no GPU is present (there is no CPU fallback).
"""
from .synth import CONFIGS, Config  # noqa: F401
