"""CPU oracle for the RTCG hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_0911_3456_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``--impl reference`` and the ``cpu_baseline`` key) may use it, and only as
the checker / the timed CPU reference -- never as a product code path.

Contents
* ``cport``    -- C restatement of the kernels rtcg-kit generates (elementwise
                 ``src/elementwise.py:204-270``, reductions
                 ``src/reduction.py:98-181``), compiled with the reference's
                 own command ``cc -O2 -ffp-contract=off -shared -fPIC``
                 (``src/jit.py:43,452-453``) and driven over the reference's
                 worker ranges with host threads (``src/elementwise.py:276-313``,
                 ``src/reduction.py:236-258``).  Same C text semantics, same
                 compiler, same libm: bit-identical to the reference.
* ``csem``     -- numpy restatement of per-element C semantics for the
                 acceptance corpus (``tests/test_acceptance.py:100-179``) and
                 tolerance helpers for float reductions.
* ``refdrive`` -- loads ``oracle/_ref/*.so`` -- the C that the reference's own
                 generator emits, compiled here by ``oracle/build_ref.py`` from
                 the reference tree -- and runs it with the reference's driver
                 semantics.  Used as the CPU baseline (kind "reference").

Pinning: ``tests/golden/*.json`` hold outputs produced by importing the
reference itself (``tests/golden/make_golden.py``); ``tests/test_oracle.py``
checks ``cport`` and ``csem`` against them, so the oracle is pinned to the
reference, not just self-consistent.
"""
