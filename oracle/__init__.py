"""TEST INFRASTRUCTURE ONLY.

CPU oracles for the CTD-S / CTD-D hot path:

* ``oracle.port``  — ctypes binding of ``oracle/libctd_oracle.so``, our plain-C
  restatement of the reference algorithm (``oracle/ctd_oracle.c``).
* ``oracle.ref``   — ctypes binding of ``oracle/_ref/libctdref.so``, the
  unmodified reference sources compiled by ``oracle/Makefile`` (present only
  where the reference was built; it travels to the GPU box as a built file).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package — and only
as the checker or as the timed CPU baseline, never as the product path.
"""
