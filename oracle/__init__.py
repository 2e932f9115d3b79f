"""CPU ORACLE for the DoGIP apply / CG hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy/SciPy fp64 code written from
/root/reference/PAPER.md (cited as P:<line>).  It shares no code with the CUDA
path (paper_1710_09913_b200/), and only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import it.
The product path must never call into this package.

Modules
  reference    exact Lagrange P_k nodes/basis on the reference simplex, B-hat
               tables (Theorem 2; Theorem 4)
  quadrature   conical-product Gauss-Jacobi rule (reading L10)
  mesh         structured simplex mesh M_N, DoF map l_T, affine maps
  coefficients material coefficient closed forms (BASELINE.json configs)
  assemble     standard FEM assembly / application of A (eq:linsys_gp P:204,
               eq:linsys_se P:335), the "definition" the DoGIP apply must equal
  dogip        the paper's DoGIP weights and Algorithm 1
               (P:491-511), used only for weight parity and check (iv)
  cg           plain conjugate gradients (reading L15)
  metrics      CSR memory model and efficiencies (eq:memory_eff,
               eq:comp_eff)

Parity pins (DESIGN.md section 3 lists one named pin per function):
tests/test_oracle_reference.py, test_oracle_tables.py, test_oracle_assemble.py,
test_oracle_cg.py and test_oracle_sampled_and_coefficients.py (the full-size
sampled-row checker ``assemble.apply_rows_sampled`` / ``mesh.cell_elements``
against the CSR route on every (d, p, form), and the coefficient closed forms:
Rodrigues rotations, the {1, 10, 100} spectrum, tanh / sin-cos point values).
Parity unpinned: only the Table 1/2 ``mem A`` column for k>=2 (coefficient-
dependent drops, reading L13), which the oracle does not claim to reproduce.
"""
