"""Oracle package -- TEST INFRASTRUCTURE ONLY (see shadowkv_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  Never imported by the product package.
"""
from .shadowkv_oracle import *  # noqa: F401,F403
