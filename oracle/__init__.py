"""CPU oracle for the linevox hot path -- test infrastructure only.

Nothing under paper_1801_01155_b200/ may import this package.  See
oracle/lvx_oracle.c for the parity status and the reference citations.
"""
