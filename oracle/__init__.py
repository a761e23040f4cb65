"""CPU oracle for the B200 path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` leg may import this package, and only as the checker or
the timed CPU baseline; the product (`paper_2203_08069_b200`) never imports
it.  Contents:

* `contractions.py` -- numpy restatement of the reference's leaf statements
  (`pkg/src/tendist/algorithms.py:80-83, 280-281, 300-301, 320, 339-340`) and
  of `sequential_evaluate` (`pkg/src/tendist/ir.py:197-229`) with its
  lexicographic accumulation order;
* `distributed.py` -- numpy restatement of `run_statement` /
  `execute` (`pkg/src/tendist/simulator.py:398-663`) at task granularity,
  used as the timed CPU path of the reference;
* `generator.py` -- numpy twin of the device input generator.

Parity is pinned against the reference's own golden values
(`pkg/tests/test_ir.py:65-112`) and against fixtures produced by running the
reference itself (`tests/golden/make_golden.py`).
"""
