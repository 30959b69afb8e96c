"""Helpers shared by the GPU tests (analytic identities used as
size-independent checks at full BASELINE sizes)."""

import math

import numpy as np


def spde_logdet(nx, ny, log_tau, log_kappa):
    """log det tau (kappa^2 I + G)^2 for the Neumann lattice Laplacian G:
    eigenvalues of G are (2 - 2cos(pi j/nx)) + (2 - 2cos(pi k/ny))."""
    lam = 2.0 - 2.0 * np.cos(np.pi * np.arange(nx) / nx)
    mu = 2.0 - 2.0 * np.cos(np.pi * np.arange(ny) / ny)
    k2 = math.exp(2.0 * log_kappa)
    return nx * ny * log_tau + 2.0 * float(np.sum(np.log(k2 + lam[None, :] + mu[:, None])))


def ar1_logdet(nt, logit_rho):
    rho = 1.0 / (1.0 + math.exp(-logit_rho))
    return -(nt - 1) * math.log(1.0 - rho * rho)


def prior_logdet(inst, theta):
    """Exact log det Q_prior(theta) of a synth instance (Kronecker identity
    log det(Q_t (x) Q_s) = n_s log det Q_t + n_t log det Q_s)."""
    spec = inst.spec
    out = spec.n_fixed * math.log(spec.fixed_prior_prec)
    for c in spec.components:
        k = c.theta_index
        if c.kind == "spde2d":
            out += spde_logdet(c.graph.nx, c.graph.ny, theta[k], theta[k + 1])
        elif c.kind == "ar1_spde2d":
            ns = c.graph.n
            out += ns * ar1_logdet(c.nt, theta[k + 2]) + c.nt * spde_logdet(
                c.graph.nx, c.graph.ny, theta[k], theta[k + 1])
        elif c.kind == "ar1":
            out += c.nt * theta[k] + ar1_logdet(c.nt, theta[k + 1])
        else:
            raise ValueError(c.kind)
    return out
