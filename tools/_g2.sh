for v in default build/var_nosep.so build/var_nocb.so build/var_nosepcb.so default; do
  if [ $v = default ]; then unset CKMPM_B200_LIB; else export CKMPM_B200_LIB=$PWD/$v; fi
  timeout 300 python tools/time_phases.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['lib'][-20:], d['prec'], 'p2g', round(d['phase_ms']['p2g'],4), 'g2p', round(d['phase_ms']['g2p'],4), 'tot', round(d['total_ms'],4))"
  PREC=4 timeout 300 python tools/time_phases.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['lib'][-20:], d['prec'], 'p2g', round(d['phase_ms']['p2g'],4), 'g2p', round(d['phase_ms']['g2p'],4), 'tot', round(d['total_ms'],4))"
done
