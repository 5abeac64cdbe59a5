"""Discontinuous Galerkin RHS / SSP-RK3 on the colored surface layout."""

from .operator import DGOperator, default_freestream, ordering_plan

__all__ = ["DGOperator", "default_freestream", "ordering_plan"]
