"""Test infrastructure: CPU oracle for the DFGT hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import
this package.  It is the checker, never the thing measured or shipped.

* ``oracle.orc``  -- the C restatement (``oracle/dfgt_oracle.c`` -> ``liboracle.so``)
* ``oracle.ref``  -- the unmodified reference compiled from /root/reference
  (``oracle/_ref/libdfgt_ref.so``; absent unless ``make -C oracle`` ran where the
  reference is mounted; the built .so travels to the GPU box).
"""
from .bindings import Oracle, Reference, load_oracle, load_reference, ORACLE_DIR  # noqa: F401
