"""CPU oracle for the GSVR hot path -- TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/gsvr/{kernels,knn,train,optim,field}.py (see
host.py and gsvr_oracle.c).  Importable only from tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs; the product package never imports it.
"""
