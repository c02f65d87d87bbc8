for v in old lib=A lib=B lib=C lib=D; do
  echo "$v c3:    $(timeout 120 python tools/gpu/kw_one.py $v 2>&1 | tail -1)"
  echo "$v c3big: $(timeout 120 python tools/gpu/kw_one.py $v c3big 2>&1 | tail -1)"
done
echo "D nopeel c3: $(SKC_KAWASE_PEEL=0 timeout 120 python tools/gpu/kw_one.py lib=D 2>&1 | tail -1)"
