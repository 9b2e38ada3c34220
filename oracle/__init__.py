"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference's algorithm for the domain-parallel
hot path (`domainpar` 0.1.0 under /root/reference/pkg/src/domainpar), used
as the checker by tests/, `__graft_entry__.smoke()` and the `cpu_baseline`
/ `--impl reference` legs of bench.py.  Nothing in the product package
(`paper_2605_11111_b200`) imports, links or calls anything in here; the
product's device path fails loudly when its CUDA extension is missing.

Parity anchoring (see tests/golden/make_golden.py and DESIGN.md §Oracle):
  * plan.py        integer planning — pinned bit-exact against integers
                   captured from the reference itself (tests/golden/plans.json)
  * conv.py        forward conv 1-D/2-D — pinned bitwise against the
                   reference's dense.conv / halo_conv outputs
                   (tests/golden/conv_*.npz); 3-D and the backward are
                   restatements (the reference has neither) pinned by
                   nested-loop and central-finite-difference tests
  * attention.py   sdpa + online softmax — pinned against reference outputs
                   (tests/golden/ring_*.npz); backward is a restatement
                   pinned by finite differences
  * sharding.py    default_chunk / redistribute layouts — pinned against the
                   reference's KATs and captured local blocks
"""
