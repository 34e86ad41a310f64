"""Cases of the oracle trajectories (tests/golden/oracle_trajectory_cfg{1,2}.npz)
where the total gradient is a cancellation residual (reading R28).

At the end of a stage the oracle's own layout sits at an equilibrium of the
interpolated dynamics: there ||g|| is a tiny fraction of the terms it is
assembled from (||g|| / sum ||term||), so no fp32 pipeline can reproduce it to
1e-4 relative, and the exact gradient differs from it by the interpolation
error of the terms, not of g.  Measured with the oracle (tests/
test_oracle_conditioning.py pins these numbers):

  cfg 1, iteration 249, stage-A multipliers: ||g|| / scale = 4.4e-8
  cfg 1, iteration 499, stage-B multipliers: ||g|| / scale = 1.6e-5

Every other (config, iteration, multipliers) case of the trajectories has
||g|| / scale >= 1e-2 (smallest: cfg 2, iteration 249, stage A, 1.1e-2) and is
held to the plain bars.  In the two cases above the bars are stated against
the term scale instead; the per-term checks (F_attr, f_field, Z against the
oracle; F_rep, g_ent against the exact gradient) apply everywhere."""

STAGE_A = (1.0, 1.2, 0.0)
STAGE_B = (1.0, 0.01, 0.6)

# (cfg, iteration, multipliers) -> measured ||g|| / scale (oracle, fp64)
CONDITIONED = {(1, 249, STAGE_A): 4.4e-8, (1, 499, STAGE_B): 1.6e-5}
COND_LIMIT = 1e-3          # a case is "conditioned" when ||g|| / scale < COND_LIMIT
