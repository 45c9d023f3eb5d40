"""CPU oracle for the sketched power method -- TEST INFRASTRUCTURE ONLY.

Nothing under ``oracle/`` is part of the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it, and only as the checker or the timed CPU
baseline -- never as the thing measured on the GPU path.

Contents
--------
``skp_oracle``      numpy/scipy restatement of the reference hot path
                    (/root/reference/pkg/src/skpower/{sketching,power,linalg}.py),
                    each function citing the reference file:line it follows.
``countsketch.c``   plain-C restatement of the PCG64 -> keys -> top-s -> signs
                    CountSketch draw (numpy 2.3.5's published algorithms), the
                    bit-exact checker for the device generator.
``gen``             seeded synthetic input recipes for BASELINE configs C1-C5.

Parity pin: ``tests/golden/make_golden.py`` imports the live reference from
/root/reference (in the build container) and writes fixtures under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks both restatements
against them.
"""
