"""CPU float64 ORACLE for the HCInfer compensated quantized linear.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
execute anything under ``oracle/``.  The product path
(``paper_2605_05819_b200`` + ``libhcinfer.so``) never imports it and shares no
code, header, table or constant generator with it.

Everything here is plain, slow and written to be checked against the paper by
eye: numpy float64, library primitives (matmul, SVD) used only as whole steps,
no blocking / fusion / reordering beyond what the defining formula states.

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n.

Modules
  packing    canonical bitstream unpack, bf16 decode              (pinned)
  quant      dequant s*(q-z), RTN quantiser                       (pinned)
  factors    truncated-SVD compensation factors                  (pinned)
  linear     compensated product y = W^x + U(Vx), stack, MoE     (pinned)
  allocate   sensitivity-aware dynamic rank allocation (App. B.1) (pinned)
  brute      brute-force / greedy optimality oracles (App. B.2)   (pinned)

No function here is "parity unpinned": each has a test in
tests/test_oracle_*.py against a closed form, a worked example printed in the
paper/SPEC (tests/golden/), an invariant, or brute force.
"""
