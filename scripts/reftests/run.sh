#!/usr/bin/env bash
# Run the reference's own test suite (/root/reference/pkg/tests, unmodified)
# against the B200 drop-in.
#
#   scripts/reftests/run.sh stage     # HERE: copy the tests into baseline/ref_tests
#                                     # (git-ignored; travels to the GPU box with gpurun)
#   scripts/reftests/run.sh run [out] # on the B200: pytest with the inthist alias plugin,
#                                     # junit xml + summary into [out] (default gpurun_out/reftests)
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
DST="$ROOT/baseline/ref_tests"
case "${1:-run}" in
  stage)
    rm -rf "$DST"; mkdir -p "$DST"
    cp /root/reference/pkg/tests/*.py "$DST/"
    sha256sum "$DST"/*.py > "$DST/SHA256SUMS"
    echo "staged $(ls "$DST"/test_*.py | wc -l) reference test files into $DST"
    ;;
  run)
    OUT="${2:-$ROOT/gpurun_out/reftests}"
    mkdir -p "$OUT"
    cd "$ROOT"
    (cd "$DST" && sha256sum -c --quiet SHA256SUMS)  # unmodified copies
    set +e
    python -m pytest -p scripts.reftests.inthist_alias "$DST" -q -rfE \
      --junitxml="$OUT/junit.xml" -p no:cacheprovider > "$OUT/pytest.txt" 2>&1
    rc=$?
    set -e
    tail -5 "$OUT/pytest.txt"
    python "$ROOT/scripts/reftests/summarize.py" "$OUT/junit.xml" > "$OUT/summary.json"
    cat "$OUT/summary.json"
    exit $rc
    ;;
  *) echo "usage: $0 stage|run [outdir]" >&2; exit 2 ;;
esac
