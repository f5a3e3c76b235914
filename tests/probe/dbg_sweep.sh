for d in 0 1 2 4 3 6 5 7; do echo "dbg=$d"; CAPSCONV_MMA_DBG=$d timeout 60 python tests/probe/run_layer.py fwd 1024,24,24,8,8,3,3,1 20; done
