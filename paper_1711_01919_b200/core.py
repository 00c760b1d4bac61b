"""Alias of `paper_1711_01919_b200.domain` under the reference's module name
(`inthist.core`), so `from inthist.core import ...` call sites keep working."""

from .domain import *  # noqa: F401,F403
