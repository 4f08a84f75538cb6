"""ORACLE — test infrastructure, NOT part of the product.

A plain, slow, obviously-correct CPU implementation of one REXII step of the
linearised rotating shallow-water equations, written from arXiv:2008.11607
(``/root/reference/PAPER.md``):

* ``oracle.coeffs`` — Appendix A table, b_m, c_{1,n}, c_{2,n}, C_{1,n}, C_{2,n},
  Gamma_n, the scalar REXI/REXII forms and the term-count rule (numpy, x87
  extended precision, rounded to fp64);
* ``oracle.lrsw`` + ``rexi_oracle.c`` — naive separable DFT, dense 3x3 complex
  Gaussian elimination per Fourier mode and pole, ascending-n accumulation,
  naive inverse DFT + Re (plain C, fp64, OpenMP over modes); the exact per-mode
  propagator and a brute-force expm for tiny grids.

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs. The CUDA product
(``paper_2008_11607_b200``) never imports, links or executes anything here, and
nothing here imports the product. The two share no kernels, headers, helpers,
tables or constant generators; only the seeded input generators
(``paper_2008_11607_b200/inputs.py``, no method arithmetic) feed both.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): the Appendix A fit defect,
Fig. 1 thresholds of the scalar form vs e^{ix}, the printed M values, the
printed max-norm errors of Tables 2-7, the exact per-mode exponential vs
scipy.linalg.expm, brute-force expm on an 8x8 grid, energy/mass conservation,
tau -> 0, linearity, the Remark 3 half-sum identity. Nothing here is
"parity unpinned".
"""
