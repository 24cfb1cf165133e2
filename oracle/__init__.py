"""CPU oracle for the PolarQuant hot path -- test infrastructure only.

``polar_oracle``  numpy restatement of the reference algorithm (bit-identical
                  to the reference on the same host; pinned by golden fixtures).
``exact``         ctypes binding of exact_oracle.c, the correctly rounded
                  float32 definition the GPU kernels implement.

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline may import
this package; the product (paper_2502_00527_b200) never does.
"""
