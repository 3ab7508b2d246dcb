"""CPU oracle for the denoise hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package, and only as the checker / the timed CPU
reference path — never as the thing shipped.  The product package
(``paper_2505_10584_b200``) never imports it.

* :mod:`oracle.schedule_oracle` — restatement of ``ditplan.inference.plan_cache``
  (``pkg/src/ditplan/inference.py:48-86``), pinned against golden vectors
  produced by the real reference (``tests/golden/make_golden.py``).
* :mod:`oracle.dit_oracle` — fp32 PyTorch-CPU restatement of the Single-DiT
  and MM-DiT denoise step, 3D RoPE, AdaLN, flow-matching Euler sampler and the
  two cache policies, from ``PAPER.md:15-17,92-136,297-316``.  The reference
  has no executable DiT, so latent parity is **unpinned** by the reference
  (SURVEY.md §8(c)); it is pinned only against this restatement.
"""
