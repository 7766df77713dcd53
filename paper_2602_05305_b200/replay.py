"""Replay the reference step driver on the B200 kernels.

The reference simulator imports its attention functions by name
(simulator.py:28-34) and calls them per (layer, head) on every diffusion step
(simulator.py:412-434, dense prefill at :317-322, verify shadow at :443-460).
Patching those names in the *caller's* namespace routes every attention
evaluation of ``run_sequence`` through libfb200.so while the reference's own
policy, KV cache, counters and unmasking stay untouched -- an end-to-end
drop-in proof.  The reference module is passed in by the caller; this
package never imports it.
"""

from __future__ import annotations

import contextlib

from . import attention as A
from . import sparse as S

PATCHED = ("attention_streamed", "attention_with_reuse", "merge_partials", "attention_dense")
SPARSE_PATCHED = {"attention_partial": A, "attention_dense": A, "merge_partials": A,
                  "build_sparse_mask": S, "sparse_attention_with_residual": S}


@contextlib.contextmanager
def patch_reference_simulator(sim_module, sparse_module=None):
    """Within the block, ``sim_module`` (flashblock.simulator) calls the
    device implementations.  Optionally also patches flashblock.sparse's
    module-level names, so measure_sparse_gap (sparse.py:225-335) builds its
    masks (K5/K6) and runs both sparse variants (K7/K8) on the device."""
    saved = {name: getattr(sim_module, name) for name in PATCHED}
    saved_sparse = {}
    try:
        for name in PATCHED:
            setattr(sim_module, name, getattr(A, name))
        if sparse_module is not None:
            for name, src in SPARSE_PATCHED.items():
                saved_sparse[name] = getattr(sparse_module, name)
                setattr(sparse_module, name, getattr(src, name))
        yield
    finally:
        for name, fn in saved.items():
            setattr(sim_module, name, fn)
        for name, fn in saved_sparse.items():
            setattr(sparse_module, name, fn)


VERIFICATION_PATCHED = ("attention_dense", "attention_partial", "attention_streamed",
                        "combine_partials", "merge_partials")


@contextlib.contextmanager
def patch_reference(pkg):
    """Route every attention evaluation of the reference package ``pkg``
    (the imported ``flashblock``) through libfb200.so: the step driver
    (simulator.py:28-34), the sparse module (sparse.py:19-25) and the
    invariant suite (verification.py:14) import the functions by name, so
    their module-level names are swapped for the device implementations.
    The reference's own policy, KV cache, counters, model and checks run
    unchanged -- its verification suite and acceptance criteria then test the
    device path."""
    saved = {name: getattr(pkg.verification, name) for name in VERIFICATION_PATCHED}
    try:
        for name in VERIFICATION_PATCHED:
            setattr(pkg.verification, name, getattr(A, name))
        with patch_reference_simulator(pkg.simulator, pkg.sparse):
            yield
    finally:
        for name, fn in saved.items():
            setattr(pkg.verification, name, fn)
