"""CPU oracle for the SpMV hot path — TEST INFRASTRUCTURE ONLY.

`spmv_oracle` restates the reference package's hot-path functions in numpy;
`c_oracle` binds the C restatement (spmv_oracle.c) for full-size checks and
the CPU baseline.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may use this package, as the checker or
the timed baseline — never as the product path.
"""
