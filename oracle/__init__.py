"""CPU oracle for the GEMV / SYMV / HEMV hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import anything from here, and only as the
checker or the CPU arm.  The product (paper_1410_1726_b200) never imports
it; its compute path is the sm_100a library and fails loudly without it.

Contents
  naive.py    numpy restatement of blockmv/reference.py (the reference's own
              oracle: wide-precision full-matrix products) plus the
              reference's input generators.
  blocked.py  numpy restatement of the reference's blocked CPU path
              (blockmv/kernels.py, offset.py, multidevice.py numerics,
              without the Kepler transaction accounting).
  streamed.c  C restatement of naive_gemv / naive_symv_hemv that streams
              column panels (never materialises the mirrored matrix) in
              wide precision with OpenMP threads: the large-N checker and
              the CPU baseline.  Built to oracle/liboracle.so.
Pinning: tests/golden/*.npz are outputs of the real reference
(`blockmv` imported from /root/reference/pkg/src by
tests/golden/make_golden.py); tests/test_oracle.py checks naive.py and
blocked.py against them bit-for-bit where the reference is deterministic,
and streamed.c against naive.py.
"""
