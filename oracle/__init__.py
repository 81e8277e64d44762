"""Parity oracle for the VLQ-ADC hot path -- TEST INFRASTRUCTURE ONLY.

* ``oracle/vlq_oracle.c`` (-> ``liboracle.so``): plain-C restatement of the
  reference search/add arithmetic, each function citing the reference line it
  follows.
* ``oracle/_ref/``: the reference implementation itself, compiled from
  /root/reference/proj by ``oracle/Makefile`` (its pybind11 module ``vlqadc``
  and the ``ref_tools`` fixture exporter).  Used to pin the restatement and as
  the ``--impl reference`` CPU arm of bench.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg
may import this package.  The product path never does.
"""
