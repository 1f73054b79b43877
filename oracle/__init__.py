"""CPU oracle for the bisector update path -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs.
The product package (paper_2407_02215_b200) never imports this.
"""

from .oracle import (OraclePool, OracleVerdict, build, lib, max_threads,  # noqa: F401
                     sum_reduce_nodes, decode_ones, decode_zeros, decode_tris)
