# A/B on the box: full GPU parity + short bench lines for the default build, then the
# same bench lines with the knob in $AB_OFF (e.g. LSQ_WALSH_DIAG=0) as the baseline.
PYEXPR="${PYEXPR_NEW:-all}" bash profiles/box_iter.sh new
echo "--- baseline ($AB_OFF)"
env $AB_OFF PYEXPR="small_configs" bash profiles/box_iter.sh base
