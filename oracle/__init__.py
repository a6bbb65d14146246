"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (fp64 for floating point) of
what the hot path of arXiv 2406.16091 computes.  It exists to prove parity of the
CUDA path and is NOT part of the product:

  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
    reference leg may import, call, link or execute anything under oracle/.
  * It shares no code with paper_2406_16091_b200/ (no kernels, headers, helpers,
    tables or constant generators) and neither side imports the other.  The
    only common input is synth/ (seeded generators with none of the method's
    arithmetic).

Modules
  reference.py   numpy: cell index (C3), counts/offsets/M_C (C4), membership (C5),
                 27-neighbourhoods (C6), O(N^2) brute-force interactions (C8-C10),
                 position update (C11), the paper's in-SM prefix sum (Listing 1).
  celllist.c     plain C, fp64 cell-list interactions (same definitions, O(N)),
                 used for the large configs and for sampled targets.
  celllist.py    ctypes loader for celllist.c (built by __graft_entry__.build()).

Every function cites the PAPER.md passage it follows (PAPER.md:L = line L of
/root/reference/PAPER.md, which does not exist on the GPU box; the citations are
for the reader).  Parity status per function is in DESIGN.md "Oracle pins".
"""
