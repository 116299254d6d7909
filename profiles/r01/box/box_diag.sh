for k in "" LSQ_TAN_ROT=0 LSQ_UNIT_CONST=0 LSQ_FOLD_DRUN=0 LSQ_WALSH_DIAG=0 LSQ_SPLIT=0; do
  echo "== $k"; env $k timeout 300 python -m pytest tests -q -m gpu -k "multipass and 5-8" 2>&1 | grep -E "passed|failed|worst" | head -3
done
