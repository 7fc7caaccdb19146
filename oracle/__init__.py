"""CPU ORACLE -- test infrastructure only.

Plain, slow, fp64 CPU implementation of what the TEM forward hot path
computes (§2.2 eq:ode/eq:expm, §3.2 eq:ratfam/eq:rkfit/eq:rmj):

* ``oracle.yee``      -- CSR assembly of K (curl-curl), M (conductivity mass)
                         and f (transmitter load) on the staggered Yee/FIT
                         edge grid (lowest-order Nedelec on a tensor hex grid,
                         lumped masses; reading R1).
* ``oracle.rkfit``    -- the shared-pole rational family of §3.2 fitted by
                         RKFIT pole relocation on a diagonal surrogate
                         (eq:rkfit), residues by linear least squares.
* ``oracle.forward``  -- per-pole sparse direct solves (K - xi_i M) x_i = f,
                         the 2 Re(S R) channel synthesis (eq:rmj), the dense
                         expm(-t M^{-1} K) b brute force (eq:expm), residual
                         and M-norm helpers.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2506_11657_b200``) never imports it and shares no code with
it; the only shared module is ``workloads`` (seeded inputs, no arithmetic).
"""
