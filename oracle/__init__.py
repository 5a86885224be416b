"""Parity oracle for the fused Harris hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker (or
as the timed CPU arm).  The product package ``paper_2212_12035_b200`` never
imports it; its GPU path fails loudly when the CUDA library is missing.

Contents
--------
* :mod:`oracle.cref`        — ctypes binding of ``liboracle_harris.so``
  (``harris_oracle.c``: f32 Appendix-B restatement and f64 sges-order
  restatement, OpenMP, thesis cbuf strip schedule).
* :mod:`oracle.npref`       — pure numpy restatement (f64 and f32), used to
  cross-check the C code and for known-answer images.
* :mod:`oracle.sges_oracle` — drives the reference package's own evaluator
  (``sges.evalref.eval_term``) on the thesis Rise program (SURVEY.md
  Appendix A); needs ``/root/reference`` (this container only).
* :mod:`oracle.synth`       — numpy mirror of the device synthetic-image
  generator, plus the tolerance metrics of SURVEY.md §8(d).
"""
