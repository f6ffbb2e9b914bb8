"""CPU oracle for the SlimFit activation-memory hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in `paper_2305_18513_b200/` imports this
package; only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may use it, and only as the checker or
the timed CPU baseline — never as the thing measured or shipped.

It is a numpy restatement (not a copy) of the reference's algorithms, each
function citing the reference `file:line` it follows (paths relative to
`/root/reference/pkg/src/slimfit/`).  Parity of the restatement itself is
pinned by `tests/golden/*.npz`, produced by `tests/golden/make_golden.py`
from the real reference package imported in the build container.
"""
