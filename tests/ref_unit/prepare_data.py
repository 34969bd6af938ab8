"""Write the fixture graphs and default.cfg the reference's tests expect
(FIXTURE_DIR / CONFIG_DIR) from the committed golden data."""
import json
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def prepare():
    data = os.path.join(HERE, "_data")
    os.makedirs(data, exist_ok=True)
    with open(os.path.join(ROOT, "tests", "golden", "fixtures.json")) as f:
        for name, text in json.load(f).items():
            with open(os.path.join(data, name + ".graph"), "w") as g:
                g.write(text)
    shutil.copy(os.path.join(ROOT, "paper_2009_10924_b200", "configs", "v100_default.cfg"),
                os.path.join(data, "default.cfg"))
    return data


if __name__ == "__main__":
    print(prepare())
