"""Alias of `paper_1711_01919_b200.formats` under the reference's module name
(`inthist.imgio`), so `from inthist.imgio import ...` call sites keep working."""

from .formats import *  # noqa: F401,F403
