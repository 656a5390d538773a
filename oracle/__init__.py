"""CPU oracle for the TMOP hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_2205_12721_b200`) imports this
package.  It may be imported only by `tests/`, by `__graft_entry__.smoke()`
and by the `cpu_baseline` / `--impl reference` legs of `bench.py`, and
there only as the checker or the timed CPU baseline -- never as the thing
measured or shipped.

`tmop_oracle` restates the reference package's algorithm
(`/root/reference/pkg/src/tmopbench`, cited file:line per function) in
vectorised numpy.  It is pinned against golden vectors produced by running
the reference itself (`tests/golden/make_golden.py`, fixtures in
`tests/golden/*.npz`) -- see `tests/test_oracle.py`.

Parity status: pinned for metrics mu_2, mu_55, mu_303 with ideal targets.
mu_7, mu_302, mu_321 do not exist in the reference: those branches are
"parity unpinned" and are checked only by finite differences, invariances
and PA-vs-FA agreement.
"""
