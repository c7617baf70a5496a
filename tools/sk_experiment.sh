# stream-K vs whole-tile decode GEMMs (tools/decode_gemm_tiled.py shapes), two processes for the env switch
for cfg in "KVPR_STREAMK=1" "KVPR_STREAMK=0"; do
  echo "== $cfg"
  env $cfg python tools/decode_gemm_tiled.py
done
