"""ORACLE -- test infrastructure only.  NOT part of the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only
as the checker (or as the timed CPU reference arm), never as the thing
measured or shipped.  The product (``paper_2310_01212_b200``) never imports
it and has no CPU execution path.

Contents:
  protocol.py     CPU restatement of the reference handshake: word codec,
                  worker state machine, per-worker trace replay
                  (/root/reference/pkg/src/persistkern/protocol.py).
                  PINNED against golden vectors generated from the reference
                  itself (tests/golden/make_golden.py -> tests/golden/*.json)
                  and, when /root/reference is present, against the live
                  reference in tests/test_oracle.py.
  work.py         numpy semantics of the payload work items.  The reference
                  has no payload arithmetic (its worker ignores `kind` and the
                  data refs, native.py:179-181), so these are the builder's
                  stated semantics: "parity unpinned" against the reference
                  for the arithmetic; protocol behaviour is pinned.
  cpu_session.py  a CPU port of the reference's thread-per-worker executor
                  (native.py:82-331), timed as the CPU baseline on the GPU box
                  (the reference cannot travel there).  Checked here against
                  the live reference's traces and timing envelope.
  projection.py   the golden per-worker write projection
                  D0 D4 (H[16+slot] D2 D1 H4 D4)* H8 of a native session.
"""
