"""CPU oracle for the pipeline-parallel stage-boundary transfer (arxiv 2602.18007).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything under
`oracle/`.  The product path (`paper_2602_18007_b200`, `libppc.so`) never imports,
links or calls it, and this package imports nothing from the product path.

Plain, slow, obviously-correct definitions, each citing the passage it follows
(P:Lnn = /root/reference/PAPER.md line, S:Lnn = SPEC.md line, BJ = BASELINE.json):

  schedule.py  O1  non-interleaved 1F1B op order per stage            (BJ)
  events.py    O2  discrete-event timing model of a 1F1B step
  transfer.py  O3  byte-level ring transfer: send/recv, header, credit
  proxy.py     O5  integer XOR stage proxy, 1F1B byte run            (harness construct)
  toy.py       O6  2-stage x 2-layer toy MLP, pipelined & un-pipelined (BJ configs[0])
  bf16.py      O7  fp32 -> bf16 round-to-nearest-even                  (BJ "1e-3 relative (bf16)")
  groups.py    a1  DCBS rank grid, groups and backend assignment
  roofline.py  O8  comm-only step roofline T* from O2                  (parity unpinned vs hardware)

Pins for every function live in tests/test_oracle_*.py (marker: not gpu).
"""
