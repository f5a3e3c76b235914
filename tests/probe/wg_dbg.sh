for d in 0 1 4 16 5 20 21; do
  echo "dbg=$d $(CAPSCONV_WG_DBG=$d timeout 60 python tests/probe/run_layer.py dK ${1:-1024,24,24,8,8,3,3,1} 10 2>&1 | tail -1)"
done
