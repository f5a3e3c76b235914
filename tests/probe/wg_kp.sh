for spec in 1024,22,22,8,16,3,3,2 1024,10,10,16,32,3,3,1; do for nq1 in 0 1; do for kp in 16 32 64 128; do
  r=$(CAPSCONV_WG_NQ1=$([ $nq1 = 1 ] && echo 1) CAPSCONV_WG_KP=$kp CAPSCONV_DEBUG=1 timeout 60 python tests/probe/run_layer.py dK $spec 10 2>&1)
  [ $nq1 = 0 ] && r=$(CAPSCONV_WG_KP=$kp CAPSCONV_DEBUG=1 timeout 60 python tests/probe/run_layer.py dK $spec 10 2>&1)
  echo "$spec nq1=$nq1 KP=$kp $(echo "$r" | grep -o 'nstg=[0-9]* stages=[0-9]*') $(echo "$r" | grep -o 'graph.*')"
done; done; done
