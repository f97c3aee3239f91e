"""Register the B200 kernel inside the reference package.

The reference resolves kernels by name only from its module-level registry
(kernels.py:276-285, ``_KERNELS`` filled by ``_registry()``), which drives
``get_kernel``/``select_kernel``/``POSPOPCNT_KERNEL`` (kernels.py:288-312),
its benchmark harness (``bench._resolve_runner``, bench.py:113-121) and its
selftest (selftest.py:44-90).  ``register(ref)`` appends a ``B200Kernel`` to
that registry without editing the reference's files, so

    pospopcnt bench --kernels b200,numba,baseline
    POSPOPCNT_KERNEL=b200 pospopcnt count FILE

run the sm_100a kernel unchanged.  (The reference's default dispatch picks
the kernel with the widest ``r``; the B200 kernel reports r=128 and so never
displaces the reference's own default unless selected by name.)
"""

from .kernels import B200Kernel


def register(ref):
    """Add the B200 kernel to the reference module ``ref`` (idempotent).

    ``ref`` is the imported reference package (``import pospopcnt``) or its
    ``kernels`` submodule.  Returns the registered kernel object.
    """
    km = getattr(ref, "kernels", ref)
    reg = km._registry()  # materialise the built-in list first (kernels.py:276)
    for k in reg:
        if getattr(k, "name", None) == B200Kernel.name:
            return k
    k = B200Kernel()
    reg.append(k)
    return k
