"""CPU oracle for the NFFT-accelerated Sinkhorn hot path (arXiv 2201.07524).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call,
link or execute anything under ``oracle/``. The product path
(``paper_2201_07524_b200``) never imports it and fails loudly if its CUDA
extension is missing.

The oracle shares no code with the CUDA path: no kernels, headers, helpers,
tables, constant generators, pre- or post-processing. The only module both
sides use is ``synthetic`` (seeded input generators, no arithmetic of the
method).

Contents (each function cites the passage it follows; P:Lx = PAPER.md line x):
  dense.py     C/OpenMP direct sums, Alg. 1 (plain and log domain), divergences
  nfft_ref.py  geometry reading, Kaiser-Bessel window, NDFT, kernel Fourier
               coefficients b_k, regularised kernel K~ with two-point Taylor K_B,
               gridding/interpolation definitions, NDFT fast summation
  exact_ot.py  exact LP optimal transport (brute force / linprog), 1-D W2 and W1 closed forms
  measures.py  entropy, KL divergence
  diagnostics.py  per-iteration residual / KL / objective trace of Alg. 1 (NEXT-3)
  laplace_ref.py  r = 1 fast summation: inner regularisation K_I, regularised kernel, NDFT far
               field + brute-force near field (NEXT-2)

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_pins.py``; none is
"parity unpinned".
"""
