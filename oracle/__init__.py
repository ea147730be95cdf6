"""CPU oracle of the BBC query path.  TEST INFRASTRUCTURE ONLY: imported by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg, never by the product
package.  Shares no code with the CUDA path (see bbc_oracle.py)."""
from . import bbc_oracle, bruteforce, sharded  # noqa: F401
