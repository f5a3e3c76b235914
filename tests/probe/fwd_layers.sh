for op in fwd dI; do for spec in 1024,24,24,8,8,3,3,1 1024,22,22,8,16,3,3,2 1024,10,10,16,32,3,3,1 1024,8,8,32,10,8,8,1; do
  timeout 60 python tests/probe/run_layer.py $op $spec 10 2>&1 | tail -1
done; done
