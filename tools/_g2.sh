tests/cpp/_bin/dropin_test jelly tests/golden/configs 12
tests/cpp/_bin/dropin_test contact tests/golden/configs
tests/cpp/_bin/dropin_test rod | tail -1
tests/cpp/_bin/dropin_test spheres | tail -1
