"""Alias of `paper_1711_01919_b200.streamed` under the reference's module name
(`inthist.streaming`), so `from inthist.streaming import ...` call sites keep working."""

from .streamed import *  # noqa: F401,F403
