"""CPU oracle for PoocH (arXiv 1907.05013) -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 NumPy implementations of what the CUDA
path computes: the CNN layer math (``layers``), the two networks and their
saved-feature-map census (``nets``), the timeline/memory simulator
(``sim``) and the keep/swap/recompute planners (``planner``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product path (``paper_1907_05013_b200``) never imports it and shares no code
with it; the only common module is ``synthdata`` (seeded random inputs).

Citations ``P:Lnnn`` are lines of PAPER.md (the paper's LaTeX source),
``S:Lnnn`` lines of SPEC.md; readings of ambiguous passages are numbered as in
DESIGN.md "Readings".
"""
