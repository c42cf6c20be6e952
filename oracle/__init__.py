"""CPU oracle for arXiv 2103.04770 (Magri, Lucarini, Lemoine, Adam, Segurado).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything under `oracle/`.  The product
path (`paper_2103_04770_b200`) never imports, calls or links this package; it shares no
code, tables or helpers with it.

Plain, slow, obviously-correct NumPy/SciPy in float64, written from PAPER.md (citations
`P:<line>`) with the readings of DESIGN.md ("A-xx" = ambiguity register of SURVEY.md 8(c)).

Modules
  spectral    discretization, frequencies, Willot/continuous symbols (P:644-645,
              A-04/A-06), unnormalised DFT pair with a naive-DFT and a scipy backend
  projection  Galerkin projection G* with mixed-control zero frequency (A-07/A-08)
  helmholtz   L^ (A-09), preconditioner M (A-11), Algorithm 2 PCG
  material    J2-Lemaitre return map (A-14/A-15), elastic, brittle (A-18)
  mech        tangent contraction, CG for G*(C:de) = -G*(sigma - Sigma)
  increment   Newton + Algorithm 1 staggered increment (A-01/A-02/A-16/A-22/A-28)

Parity-pin status per function is stated in each module header; nothing here is
"parity unpinned" except the full post-peak load curves (A-27), see DESIGN.md.
"""
