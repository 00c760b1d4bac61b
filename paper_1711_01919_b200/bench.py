"""Alias of `paper_1711_01919_b200.harness` under the reference's module name
(`inthist.bench`): BenchConfig, run_bench, write_csv, synth_image, tensor_checksum."""

from .harness import *  # noqa: F401,F403
from .harness import (CSV_HEADER, BenchConfig, BenchRecord, csv_text, run_bench,  # noqa: F401
                      run_window_sensitivity, synth_image, tensor_checksum, write_csv)
