#!/bin/bash
# Stage the reference's own test suite (unmodified) for a run against this
# package through the `pmewald` alias (tools/ref_suite/pmewald).  Output:
# baseline/_ref_suite/ (git-ignored; travels to the GPU box with gpurun):
#   tests/        the reference's pkg/tests/*.py, unmodified
#   _ref_modules/ the reference's oracle.py and cli.py (validation oracles
#                 and CLI front end, out of the product's scope; test
#                 infrastructure only)
#   pmewald/      the alias package
# Run (GPU box):  bash baseline/_ref_suite/run.sh
set -e
REF=${REF:-/root/reference/pkg}
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
OUT=$ROOT/baseline/_ref_suite
rm -rf "$OUT" && mkdir -p "$OUT/tests" "$OUT/_ref_modules"
cp "$REF"/tests/*.py "$OUT/tests/"
cp "$REF"/src/pmewald/oracle.py "$REF"/src/pmewald/cli.py "$OUT/_ref_modules/"
cp -r "$ROOT/tools/ref_suite/pmewald" "$OUT/pmewald"
cat > "$OUT/run.sh" <<'EOS'
#!/bin/bash
# the reference's 190 tests against paper_1712_04732_b200 via the pmewald alias
cd "$(dirname "$0")"
export PMEWALD_REF_STAGED=$PWD/_ref_modules
export SE_B200_DETERMINISTIC=1
export PYTHONPATH=$PWD:$PWD/../..${PYTHONPATH:+:$PYTHONPATH}
python -m pytest tests -q -p no:cacheprovider -rf "$@"
EOS
chmod +x "$OUT/run.sh"
echo "staged $(ls "$OUT/tests" | wc -l) test files into $OUT"
