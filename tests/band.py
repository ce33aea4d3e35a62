"""SURVEY §8(c) decision-band parity rule (test infrastructure).

Two cost terms are discontinuous in the state: manipulability jumps from 0 to
1 - m where m crosses k_m (costs.py:126-127), and world collision is a strict
inequality on the clearance (kernels/jit.py:316,326). An FP32 rollout whose
positions differ from the float64 reference by ~1e-6 may take the other
branch for an entry that sits within rounding of the switch point. The rule:

  1. the oracle reports each entry's margin (m - k_m, clearance - radius);
  2. an entry with |margin| < BAND may take either branch: where the device
     took the other one, substitute the reference's branch (the term value
     and, through the weights, the step cost and the discounted total);
  3. count those substitutions (band hits) and report them;
  4. every other entry must agree: zero out-of-band flips, and the corrected
     totals must pass the weight-safe check.

The policy update of a step with band substitutions is re-derived from the
corrected totals and the device's own controls (oracle arithmetic), and that
command is what is compared with the reference's; the device's command is
checked for consistency with its own totals.
"""

from __future__ import annotations

import numpy as np

BAND = 1e-5


def weight_safe(tot, ref_tot, ref_w, beta, tol):
    """|d(c_i - c_min)| <= tol*beta for every particle whose reference weight > 1e-6."""
    ok = np.isfinite(ref_tot)
    assert np.array_equal(np.isfinite(tot), ok), "quarantine sets differ"
    rel_gpu = tot[ok] - tot[ok].min()
    rel_ref = ref_tot[ok] - ref_tot[ok].min()
    sel = ref_w[ok] > 1e-6
    err = float(np.abs(rel_gpu - rel_ref)[sel].max())
    assert err <= tol * beta, err
    return err


def apply_bands(gpu_terms, ref_terms, margins, weights, gamma, terminal_weight, band=BAND,
                term_tol=(1e-4, 2e-4)):
    """Compare the device's per-term arrays (n,H) with the reference's under
    the band rule. Returns (step-cost correction (n,H), total correction (n,),
    report dict). Raises AssertionError on an out-of-band disagreement."""
    rtol, atol = term_tol
    report = {"manip_band_hits": 0, "envcoll_band_hits": 0}
    n, H = next(iter(ref_terms.values())).shape
    dstep = np.zeros((n, H))
    scale = {"manip": weights.alpha_manip, "envcoll": weights.alpha_coll}
    for term, key in (("manip", "manip"), ("envcoll", "env")):
        if term not in ref_terms:
            continue
        g, r = np.asarray(gpu_terms[term]), np.asarray(ref_terms[term])
        m = np.asarray(margins.get(key, np.full((n, H), np.inf)))
        in_band = np.abs(m) < band
        if term == "envcoll":
            differs = g != r
        else:  # a branch flip: one side zero, the other 1 - m > 0
            differs = (g == 0.0) != (r == 0.0)
        flips_out = differs & ~in_band
        assert not flips_out.any(), (
            f"{term}: {int(flips_out.sum())} out-of-band branch flips, e.g. at "
            f"{np.argwhere(flips_out)[:3].tolist()} margins {m[flips_out][:3]}")
        sub = differs & in_band
        report[f"{term}_band_entries"] = int(in_band.sum())
        report[f"{term}_flips"] = int(differs.sum())
        report[f"{term}_band_hits"] = int(sub.sum())
        dstep += np.where(sub, scale[term] * (r - g), 0.0)
        same = ~sub
        np.testing.assert_allclose(g[same], r[same], rtol=rtol, atol=atol, err_msg=term)
    for term in ("pose", "stop", "joint", "selfcoll"):
        if term not in ref_terms:
            continue
        np.testing.assert_allclose(gpu_terms[term], ref_terms[term], rtol=rtol, atol=atol, err_msg=term)
    disc = gamma ** np.arange(H)
    disc[-1] *= terminal_weight
    dtot = dstep @ disc
    return dstep, dtot, report


def corrected_command(controls, totals, means_in, variances_in, beta, alpha_mu, alpha_sigma, smin, smax,
                      isotropic=False):
    """Command and policy of one iteration from given totals and controls
    (policy.py:103-155, oracle arithmetic), starting from the shifted policy."""
    from oracle import mppi_oracle as O

    w = O.weights_from_totals(totals, beta)
    mu, var = O.blend_policy(means_in, variances_in, controls, w, alpha_mu, alpha_sigma, smin, smax, isotropic)
    return mu[0].copy(), mu, var, w
