"""Instance CSV (data.cpp:203-271) round trip and refusals — the reference's
test_data.cpp:310-336 cases, through the host-side mirror (no device)."""
import numpy as np
import pytest

from paper_2605_30267_b200 import ot


def test_round_trip_is_exact(tmp_path):
    a, b, Cm = ot.synthetic_instance(3, 4, 99)
    p = ot.with_epsilon(ot.make_problem(a, b, Cm, 1.0), 0.037)
    f = tmp_path / "instance.csv"
    ot.write_instance_csv(f, p)
    q = ot.read_instance_csv(f)
    assert q.n() == 3 and q.m() == 4 and q.epsilon == p.epsilon
    assert np.array_equal(q.a, p.a) and np.array_equal(q.b, p.b) and np.array_equal(q.C, p.C)


def test_rescaled_problem_writes_the_solver_unit_cost(tmp_path):
    a, b, Cm = ot.synthetic_instance(5, 3, 7)
    p = ot.rescale_problem(ot.make_problem(a, b, Cm, 0.05))
    f = tmp_path / "r.csv"
    ot.write_instance_csv(f, p)
    q = ot.read_instance_csv(f)
    assert q.epsilon == 1.0 and np.array_equal(q.C, Cm / 0.05)


@pytest.mark.parametrize("text", ["nope\n", "name,index,value\nn,0,2\n",
                                  "name,index,value\nn,0,1\nm,0,1\nepsilon,0,1\na,1,1\n",
                                  "name,index,value\nn,0,1\nm,0,1\nepsilon,0,1\nz,0,1\n",
                                  "name,index,value\nn 0 1\n"])
def test_malformed_files_are_refused(tmp_path, text):
    f = tmp_path / "bad.csv"
    f.write_text(text)
    with pytest.raises(ot.MalformedLine):
        ot.read_instance_csv(f)


def test_missing_file_is_an_io_error(tmp_path):
    with pytest.raises(ot.IoError):
        ot.read_instance_csv(tmp_path / "absent.csv")
