for lib in /tmp/libpp_default.so tools/libpp_640_1.so; do
  cp $lib paper_1907_13257_b200/libpp.so
  echo "### $lib"
  for w in inception_v3 gnmt biglstm; do for M in 2 4 8; do
    PP_VERBOSE=1 timeout 120 python bench.py --workload $w --M $M --no-cpu-baseline --steps 2 --warmup 1 --rounds 2 2>&1 >/dev/null | grep "pp: M" | sort | uniq -c | head -2 | sed "s/^/$w /"
  done; done
done
