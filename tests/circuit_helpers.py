"""Circuit builders shared by the GPU parity tests and the CPU race check."""


def random_circuit(rng, n, nlayers):
    """Random layered circuit over every gate kind, pattern and role (built here; the pinned
    oracle is the reference for it)."""
    from paper_2506_04891_b200.circuits import Circuit, Layer, Role, all_qubits, chain_pairs, explicit, ring_pairs
    from paper_2506_04891_b200.gates import GATE_TRAITS

    kinds = list(GATE_TRAITS)
    layers = []
    for _ in range(nlayers):
        g = kinds[rng.integers(len(kinds))]
        tr = GATE_TRAITS[g]
        if tr.arity == 1:
            pat = all_qubits() if rng.random() < 0.6 else explicit(*[(int(w),) for w in rng.choice(n, 3, replace=False)])
        else:
            r = rng.random()
            if r < 0.35:
                pat = chain_pairs()
            elif r < 0.7:
                pat = ring_pairs()
            else:
                pat = explicit(*[tuple(int(w) for w in rng.choice(n, 2, replace=False)) for _ in range(3)])
        if tr.param_count == 0:
            layers.append(Layer(g, pat))
            continue
        role = [Role.TRAINABLE, Role.ENCODING, Role.FIXED][rng.integers(3)]
        if role is Role.FIXED:
            npos = n if pat.kind.value == "all" else (n - 1 if pat.kind.value == "chain" else
                                                        (n if pat.kind.value == "ring" else len(pat.wires)))
            vals = rng.uniform(-3, 3, (npos, tr.param_count)).tolist()
            layers.append(Layer(g, pat, role, vals))
        else:
            layers.append(Layer(g, pat, role))
    return Circuit(n, layers)
