"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no scheduling, no edge-cost
conversion, no projection): it only builds DFG descriptors (op times in ps,
edge bytes, memory and parameter bytes, link parameters) and epochs-vs-batch
curves, following the recipe in DESIGN.md §Inputs (reading
R20 for the analytic cost model of PAPER.md:511).
"""
from .dfgs import (toy12, gnmt, biglstm, inception_v3, random_dag, chain, star,
                   independent, diamond, PAPER_PROFILE, B200_PROFILE)
from .curves import (toy12_scenario, sweep_scenario, inception_fixture, biglstm_fixture,
                     gnmt_fixture)

__all__ = ["toy12", "gnmt", "biglstm", "inception_v3", "random_dag", "chain", "star",
           "independent", "diamond", "PAPER_PROFILE", "B200_PROFILE", "toy12_scenario",
           "sweep_scenario", "inception_fixture", "biglstm_fixture", "gnmt_fixture"]
