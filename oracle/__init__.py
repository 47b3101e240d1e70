"""PGT-I float64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import anything from this package.  The product
path (``paper_2507_11683_b200``) never imports it and shares no code with it:
the only module both sides read is ``synth`` (seeded raw inputs, none of the
method's arithmetic).

It is the plain definition of what the index-batched training step computes
(PAPER.md = "P:n"; SPEC.md = "S:n"):

* ``windows``      -- window count, 70/10/20 split, Alg. 1 literal:
                      stack every snapshot, scalar mu/sigma over x_train,
                      standardise x and y (the fp32 formula of reading c9/O4).
* ``memory``       -- Eq. 1 and Eq. 2, generalised to
                      T_in != T_out, plus the halo-shard size (O14).
* ``philox``       -- Philox4x32-10 (Salmon et al., Random123) and the
                      per-epoch index plan of reading c16/O6.
* ``transitions``  -- P_f = D_O^-1 A, P_b = D_I^-1 A^T (Li et al. Eq. 2 [ext],
                      reading c1/c4/c5).
* ``dcgru``        -- stepwise stacked DCGRU forward (reading c1-c7),
                      MAE loss, hand-written reverse mode.
* ``adam``         -- torch-default Adam in float64 (reading c21).
* ``ddp``          -- gradient mean over ranks in ascending order.

Every function cites the passage it follows.  Functions whose result is not
pinned by any independent check say "parity unpinned" (none at present; see
DESIGN.md "Oracle pins").
"""
