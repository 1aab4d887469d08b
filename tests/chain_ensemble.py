"""Reading Q28 for a recycle chain: the spaces a chain hands on
depend on rounding (their trailing, ill-determined directions), so a chain
run by the GPU is judged per system against chains of the oracle run on the
same sequence with b perturbed by relative 1e-15 (seeded), not against one
oracle chain.  Test infrastructure (calls only oracle/ and synth/)."""
import numpy as np

from oracle.sequence import run_sequence


def oracle_chain_counts(cfg, items, runs=5, seed=77):
    """Iteration counts per system: row 0 the unperturbed oracle chain, then
    `runs` perturbed chains."""
    rng = np.random.default_rng(seed)
    ens = [[r.iterations for r in run_sequence(cfg, items)]]
    for _ in range(runs):
        pert = [dict(it, b=it["b"] * (1 + 1e-15 * rng.standard_normal(it["b"].shape)))
                for it in items]
        ens.append([r.iterations for r in run_sequence(cfg, pert)])
    return np.array(ens)


def within_ensemble(its, ens):
    """Each count inside [min, max] of its column widened by max(2, 3 %)
    (BASELINE's iteration criterion applied to the ensemble's ends)."""
    for j, m in enumerate(its):
        lo, hi = ens[:, j].min(), ens[:, j].max()
        if not lo - max(2, 0.03 * lo) <= m <= hi + max(2, 0.03 * hi):
            return False, (j, list(its), list(ens[:, j]))
    return True, None
