# usage: ab.sh ENVVAR VAL_A VAL_B op spec...   (alternates A/B twice)
var=$1; a=$2; b=$3; shift 3
for rep in 1 2; do for v in $a $b; do for os in "$@"; do
  op=${os%%:*}; spec=${os#*:}
  echo "$var=$v $(env $var=$v timeout 60 python tests/probe/run_layer.py $op $spec 10 2>&1 | tail -1)"
done; done; done
