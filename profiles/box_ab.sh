bash profiles/box_iter.sh new
echo "--- baseline (LSQ_SKIP_EMPTY=0)"
LSQ_SKIP_EMPTY=0 PYK="-k small_configs" bash profiles/box_iter.sh base
