"""Alias of `paper_1711_01919_b200.matching` under the reference's module name
(`inthist.likelihood`), so `from inthist.likelihood import ...` call sites keep working."""

from .matching import *  # noqa: F401,F403
