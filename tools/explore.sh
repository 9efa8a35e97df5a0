export LYAP_VERBOSE=1
for spec in "$@"; do
  tag=$(echo $spec | tr ' :' '__')
  timeout 900 python tools/explore_cfg.py $spec > gpurun_out/explore_$tag.log 2>&1; echo "$spec rc=$?"
done
