# pass GB/s at one config for env variants: VARIANTS="name:ENV=1+ENV2=2 ..."
C=${CONFIG:-all128}; N=${NCOLS:-512}
for v in $VARIANTS; do
  name=${v%%:*}; envs=${v#*:}
  env $(echo $envs | tr '+' ' ') timeout 600 python tools/pass_bench.py $C $N 1 2>&1 | tail -1 | sed "s/^/$name /"
done
