"""Alias of `paper_1711_01919_b200.compute` under the reference's module name
(`inthist.strategies`), so `from inthist.strategies import ...` call sites keep working."""

from .compute import *  # noqa: F401,F403
