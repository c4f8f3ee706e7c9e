"""CPU oracle for the hierarchical ZeRO++ (hpZ + qwZ + qgZ) data-parallel hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2501_04266_b200`` + ``libhz.so``) never
imports it and has no CPU fallback.

The oracle is written from the paper (arXiv 2501.04266, ``PAPER.md``; cited as
``P:<line>``) and from the readings listed in ``DESIGN.md`` §3 where the paper is
silent.  It is plain NumPy (fp32 where the method's arithmetic is fp32, because
north_star fixes fp32 scales and a floating-point value decides each integer
code; fp64 only for the brute-force error references in the tests).  It
simulates every rank of the hierarchy in one process, as a sequential program,
and shares no code, header, table or constant generator with the CUDA path.

Modules
  quant        O4-O6  block quantize / pack / dequantize
  partition    O1-O3  rank digits, padding, digit-reversed map    (Table IV)
  collectives  O7-O9  hierarchical qwZ/hpZ all-gather, qgZ RS
  volume       O10    closed-form communication volumes           (Tables VII, VIII)

Pins: every function is pinned in ``tests/test_oracle_*.py`` against values or
properties fixed by the paper / SPEC worked examples / mathematics, never by
re-running its own formula.  No function here is "parity unpinned".
"""

from . import quant, partition, collectives, volume  # noqa: F401
