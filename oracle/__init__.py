"""CPU oracle for the moeplace hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package, and only as the checker / the timed CPU
baseline.  The product (``paper_2508_09229_b200`` / ``moeplace``) never imports it: the product
path has no CPU fallback.

What it is: a restatement, in numpy + numba (the reference package's declared dependencies,
/root/reference/pkg/pyproject.toml:10-13), of the operations SPEC.md specifies for the path:
  gen.py       generate_trace            SPEC.md:123-131, 166 (+ our counter-based sampler)
  stats.py     estimate_frequencies
  evaluate.py  token_hops / evaluate / objective_value / gain / communication_map
                                          SPEC.md:336-379, 381-390
  topology.py  all_pairs_hops (BFS), cost_matrix, build_instance coefficients
                                          SPEC.md:51-59, 198-206, 273-281, 308

Parity pinning: the reference ships NO implementation (SPEC + paper + errors.py only; see
SURVEY.md §0), so there is no reference binary or Python module to run and no reference test
suite.  The oracle is pinned instead to every known-answer example SPEC.md gives for these
operations (SPEC.md:48-59, 129-131, 137-139, 146-148, 155-157, 204-206, 279-281, 342-344,
350-353, 359-361, 368-370, 377-379), the acceptance criteria SPEC.md:445-453 and the 48 gain
cells of PAPER.md Tables 2-4; tests/golden/ holds those vectors and the script that made them.
Independent cross-oracles where they exist in this container: networkx / scipy.sparse.csgraph
(BFS), numpy.bincount (histograms), scipy.optimize.milp (solver).
"""
