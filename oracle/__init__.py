"""CPU fp64 oracle for the space-time multigrid of arXiv:1911.09548.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1911_09548_b200``) never imports it and
shares no code with it: the oracle re-derives every operator from the paper
(PAPER.md line numbers cited per function) in plain numpy / scipy.sparse, with
no blocking, fusion or reordering beyond what the definitions state.

Modules
  mesh       structured hex (3D) / quad (2D) meshes, edge enumeration, coarsening
  fem        lowest-order Nedelec mass M_sigma, curl-curl K_nu, nodal K_n, G, P_edge
  time_dg    dG(q) time matrices (q = 0 is the paper's implicit Euler, Eq. (1))
  spacetime  L_{tau,h}, smoother S (Eq. 2), nodal correction A (Eq. 5)
  multigrid  coarsening rule (Eq. 3), hierarchy, V-cycle, solve
  lfa        scalar test-equation (Eq. 4) two-grid analysis

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``; see DESIGN.md section "Oracle pins".
"""
