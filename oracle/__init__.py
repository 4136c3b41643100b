"""CPU ORACLE -- test / baseline infrastructure only.

`oracle.Oracle` wraps the plain-C restatement (oracle/sk_oracle.c); `oracle.Ref`
wraps the reference itself compiled from /root/reference (oracle/_ref). Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
may import this package. The product package never does.
"""
from .oracle import (Oracle, Ref, OracleState, RefState, build, openblas, ref_available, scipy_lapack,  # noqa: F401,E501
                     oracle_available)
